/*
 * deepinverse.h -- C ABI of the B200-native DeepInverse batched signal-recovery library.
 *
 * The library computes, for every image b of a batch, the DeepInverse map
 *     x_hat_b = M(y_b, Omega)                                   (§4)
 * from measurements y_b = Phi x_b in R^M (§1) with Phi fixed:
 *   1. lifting layer   x_tilde = Phi^T y, viewed as n1 x n2 row-major
 *   2. conv layer 1    64 filters 11x11x1  + bias + ReLU, crop S        (Eq. (1))
 *   3. conv layer 2    32 filters 11x11x64 + bias + ReLU, crop S
 *   4. conv layer 3     1 filter  11x11x32 + bias (+ ReLU iff DI_FLAG_FINAL_RELU)
 * Each layer is the full (n+10)x(n+10) convolution of Eq. (1) cropped back to n1 x n2 by S, which
 * equals a 'same' zero-padded cross-correlation with the spatially flipped kernel.
 *
 * Every step runs in hand-written sm_100a CUDA kernels.  There is no CPU path: a context can only be
 * created on a compute-capability-10.0 device, otherwise DI_ERR_DEVICE.
 *
 * Threading: calls on different contexts are independent.  One context serves one in-flight
 * di_recover at a time (it owns a single workspace).  Error details are thread-local.
 */
#ifndef DEEPINVERSE_H_
#define DEEPINVERSE_H_

#ifdef __cplusplus
extern "C" {
#endif

typedef struct di_ctx_s* di_ctx;

typedef enum {
  DI_OK = 0,
  DI_ERR_ARG = 1,    /* null pointer, batch out of [1, max_batch], unknown enum / flag        */
  DI_ERR_DIM = 2,    /* ldy < m, bad leading dimension or alignment                           */
  DI_ERR_DOMAIN = 3, /* m < 1, m > N = n1*n2, n1 or n2 < 1                     */
  DI_ERR_DEVICE = 4, /* no CUDA device, or device is not sm_100 (compute capability 10.0)     */
  DI_ERR_OOM = 5,    /* device or pinned-host allocation failed                               */
  DI_ERR_CUDA = 6    /* a CUDA runtime / driver call or kernel launch failed                  */
} di_status;

typedef enum {
  DI_PREC_FP32 = 0, /* fp32 storage, fp32 FFMA arithmetic (SIMT): parity <= 1e-5 rel-L2           */
  DI_PREC_TF32 = 1, /* fp32 storage, TF32 tensor-core products, fp32 accumulation                  */
  DI_PREC_BF16 = 2  /* bf16 storage of Phi, y, Omega and x_tilde/h1/h2; fp32 accumulation; tcgen05 */
} di_precision;

typedef enum { DI_DTYPE_F32 = 0, DI_DTYPE_BF16 = 1 } di_dtype;

enum {
  DI_FLAG_XCORR = 1u << 0,        /* taps given in cross-correlation (torch) convention; default: the true
                                     convolution of Eq. (1) (reading Q2)           */
  DI_FLAG_FULLMAP_BIAS = 1u << 1, /* b_l given as [C_out][n1+10][n2+10]; default: [C_out] */
  DI_FLAG_FINAL_RELU = 1u << 2    /* ReLU after layer 3 (PAPER.md:118 read literally); default off       */
};

/* One layer of a custom stack ("DeepInverses with larger capacities"):
 * an Eq. (1) layer with 11x11 taps, W [cout][cin][11][11] (orientation per DI_FLAG_XCORR), b [cout] per channel
 * (NULL = zero).  ReLU after every layer but the last (the last one iff DI_FLAG_FINAL_RELU), as in Eq. (1). */
typedef struct {
  int cin, cout;
  const float* w;
  const float* b;
} di_layer;

/* Arguments of di_create.  All pointers are HOST pointers; di_create deep-copies them and the caller may
 * free them on return.  Weight layout [C_out][C_in][11][11] row-major fp32; biases fp32,
 * layout per DI_FLAG_FULLMAP_BIAS; a NULL bias pointer means zero biases.  In DI_PREC_BF16 mode Phi and
 * the weights are rounded to bf16 (round-to-nearest-even); biases stay fp32. */
typedef struct {
  int m;                 /* measurements M, 1 <= m <= n1*n2                                   */
  int n1, n2;            /* image rows / columns, N = n1*n2                                   */
  const void* phi;       /* Phi [m][n1*n2] row-major, dtype phi_dtype           */
  di_dtype phi_dtype;
  const float* w1;       /* [64][1][11][11]  */
  const float* b1;
  const float* w2;       /* [32][64][11][11] */
  const float* b2;
  const float* w3;       /* [1][32][11][11]  */
  const float* b3;
  di_precision precision;
  unsigned flags;        /* DI_FLAG_*                                                         */
  int device;            /* CUDA device ordinal                                               */
  int max_batch;         /* largest batch of a single di_recover call; sizes the workspace    */
  const float* lift;     /* optional learned lifting matrix L [n1*n2][m] row-major fp32: x_tilde = L y
                            ("one could learn the weights").  NULL: the
                            paper's fixed adjoint L = Phi^T.  Phi still defines di_measure.   */
  int n_layers;          /* 0: the paper's three layers w1..b3.  >= 2: the custom stack `layers` (w1..b3 unused):
                            layers[0].cin = 1, layers[n-1].cout = 1, layers[i].cin = layers[i-1].cout.  Supported
                            (FP32, TF32 and BF16 contexts, per-channel biases): first layer 1 -> {32, 64},
                            interior layers {32, 64} -> {32, 64} (FP32 and BF16 also
                            128 on either side: "larger capacity"), last layer 32 -> 1; TF32 also needs
                            n2 % 4 == 0.  Other shapes or DI_FLAG_FULLMAP_BIAS: DI_ERR_ARG.  Custom stacks support
                            di_recover / di_recover_host / di_recover_from_proxy / sensing / metrics and training
                            (per-channel or zero biases); di_debug_stage stages >= 1 are for the paper's stack
                            only (DI_ERR_ARG).                                                                   */
  const di_layer* layers;
} di_create_args;

/* Create a context on args->device.  On failure *out is set to NULL and a status is returned. */
di_status di_create(const di_create_args* args, di_ctx* out);

/* Recover a batch, asynchronously on `stream` (a cudaStream_t; NULL = legacy default stream).
 *   y:    DEVICE pointer, [batch][ldy] row-major; element type fp32 for FP32/TF32, bf16 for BF16;
 *         only the first m entries of each row are read.  ldy >= m.
 *   xhat: DEVICE pointer, [batch][n1][n2] fp32, written.
 * Both stay owned by the caller and must remain valid until the stream work completes.
 * Argument errors are reported synchronously before any work is enqueued; launch failures as
 * DI_ERR_CUDA.  No host synchronisation happens inside. */
di_status di_recover(di_ctx ctx, const void* y, long long ldy, int batch, float* xhat, void* stream);

/* ---- Row-sharded Phi (PAPER.md:148, 181 -- images beyond one GPU's Phi) -------------
 * With Phi split over its M rows across G ranks (rank g holds Phi_g = rows [lo_g, hi_g) and the matching entries
 * y_g of every measurement), the lifting layer is a sum of per-rank partials:
 *     x_tilde_b = Phi^T y_b = sum_g Phi_g^T y_{g,b}.
 * A context created with Phi_g (m = hi_g - lo_g rows; any 1 <= m <= N) computes its partial with
 * di_proxy_partial; the caller sums the partials across ranks (one NCCL reduce-scatter over the batch, or an
 * all-reduce) and runs the convolutions on the summed proxy with di_recover_from_proxy.
 *   di_proxy_partial:      y DEVICE [batch][ldy] (di_recover's element type), xt_part DEVICE [batch][n1*n2] fp32,
 *                          written (fp32 even in BF16 contexts: partials are summed before any rounding).
 *   di_recover_from_proxy: xt DEVICE [batch][n1*n2] fp32 (read; BF16 contexts round it once, RNE, to the bf16
 *                          x_tilde), xhat DEVICE [batch][n1][n2] fp32 (written).  Uses the context's workspace.
 * Errors as di_recover.  Learned-lifting contexts (args->lift) apply L's rows in place of Phi_g^T. */
di_status di_proxy_partial(di_ctx ctx, const void* y, long long ldy, int batch, float* xt_part, void* stream);
di_status di_recover_from_proxy(di_ctx ctx, const float* xt, int batch, float* xhat, void* stream);

/* The same reduce-scatter done by the lifting GEMM itself over peer memory: rank `rank` of `world` (<= 8) computes its
 * fp32 partial for all `batch` images (batch % world == 0, nb = batch / world) and its epilogue stores the rows of
 * image b straight into slot `rank` of the staging buffer of b's owner r = b / nb:
 *     slots[r] + (rank * nb + b % nb) * n1*n2        (slots[r]: DEVICE pointer usable on this GPU -- the owner's
 *                                                      staging [world][nb][n1*n2] fp32, peer-mapped for r != rank)
 * After every rank's di_proxy_scatter has completed (a cross-rank barrier, the caller's), each owner runs
 * di_recover_from_slots on its staging: x_tilde = sum of the world slots in rank order (deterministic; rounded once
 * to bf16 in BF16 contexts), then the convolutions, x_hat DEVICE [nb][n1][n2] fp32.  FP32 contexts compute the
 * partial locally and copy its rows out.  Errors as di_recover (world / rank / divisibility: DI_ERR_ARG). */
di_status di_proxy_scatter(di_ctx ctx, const void* y, long long ldy, int batch, float* const* slots, int world,
                           int rank, void* stream);
di_status di_recover_from_slots(di_ctx ctx, const float* staging, int world, int nb, float* xhat, void* stream);

/* End-to-end variant with HOST buffers: copies y (host, pinned or pageable) to the device, recovers, copies
 * x_hat back to `xhat_host` (pinned host memory makes the copies asynchronous).  Kernels run on `stream`; batches
 * >= 512 are split into chunks shrinking 4x (3B/4, 3B/16, ..., the last >= 128 images) whose x_hat copies run on an
 * internal stream, overlapping the next chunk's kernels.  Returns after all work and copies have completed.  Results equal di_recover's bit for bit (every
 * image is computed independently of the batch composition). */
di_status di_recover_host(di_ctx ctx, const void* y_host, long long ldy, int batch, float* xhat_host,
                          void* stream);

/* ---- Sensing model and metrics around the recovery path --------------------------------
 * di_measure:   y = Phi x (§1) for a batch of images with the context's Phi.
 *               x: DEVICE [batch][n1][n2] fp32 (row-major vectorisation j = r*n2 + c, Q8);
 *               y: DEVICE [batch][ldy], storage type of the precision (bf16 for BF16: x and Phi as bf16, fp32
 *               accumulation, one RNE rounding; fp32 for FP32/TF32).  ldy >= m.  Asynchronous on `stream`.
 * di_add_noise: y_b += w_b with w_b ~ N(0, sigma_b^2 I), sigma_b^2 = ||y_b||^2 / (m * 10^(snr_db/10)), i.e.
 *               10 log10(||y||^2 / E||w||^2) = snr_db (Table 3's 20 dB noise; measurement-domain
 *               reading DESIGN.md Q14).  Standard normal i of image b is counter b*m + i of the splitmix64/Box-Muller
 *               stream keyed by (seed, stream 5) -- the generator of synth/rng.py.  snr_db = +inf: no-op.
 *               y: DEVICE, storage type, in place.
 * di_metrics:   per image, fp64: out[b] = PSNR = 10 log10(max(x_b)^2 / MSE) (+inf if MSE = 0),
 *               out[batch + b] = NMSE = ||xhat_b - x_b||^2 / ||x_b||^2, out[2*batch + b] = success
 *               1(NMSE <= 0.1).  xhat, x: DEVICE [batch][n1][n2] fp32; out: DEVICE [3][batch] double.
 * batch must lie in [1, max_batch] (di_measure / di_add_noise) or >= 1 (di_metrics). */
di_status di_measure(di_ctx ctx, const float* x, int batch, void* y, long long ldy, void* stream);
di_status di_add_noise(di_ctx ctx, void* y, long long ldy, int batch, double snr_db, unsigned long long seed,
                       void* stream);
di_status di_metrics(di_ctx ctx, const float* xhat, const float* x, int batch, double* out, void* stream);
/* di_recover_metrics: di_recover followed by di_metrics on the same batch (the Monte-Carlo loop of PAPER.md:159-160,
 *               Figs. 2-4).  By default the metrics are the separate di_metrics pass; a context created with the
 *               environment variable DI_EXP_FUSED_METRICS=1 computes them inside conv layer 3's epilogue on the BF16
 *               path instead (each output compared with x_true as it is written; per-item fp64 partials combined in
 *               a fixed order, deterministic) -- measured slower on B200.  y, ldy, batch, xhat: as
 *               di_recover; x_true: DEVICE [batch][n1][n2] fp32 ground truth; metrics: DEVICE [3][batch] double as
 *               di_metrics.  Errors as di_recover; DI_ERR_ARG if x_true or metrics is NULL. */
di_status di_recover_metrics(di_ctx ctx, const void* y, long long ldy, int batch, const float* x_true, float* xhat,
                             double* metrics, void* stream);

/* ---- Training step (contexts of the paper's stack with per-channel or zero biases) ----------
 * FP32 contexts: SIMT forward and backward (fp32 products).  TF32 contexts: TF32 tensor-core forward; backward on the
 * tensor cores with bf16 operands for the layer-2 data / weight gradients and the thin-layer weight gradients, TF32
 * for the layer-3 data gradient.  BF16 contexts: the bf16 forward (weights = RNE-rounded fp32 master parameters),
 * the same tensor-core backward; BF16 training needs n2 % 4 == 0 (DI_ERR_ARG otherwise).  Gradients and the
 * parameters stay fp32.
 * Parameter vector layout (di_num_params() = 259 521 floats), the orientation given to di_create (true convolution,
 * or cross-correlation with DI_FLAG_XCORR):  [W1 64x1x11x11 | W2 32x64x11x11 | W3 1x32x11x11 | b1 64 | b2 32 | b3 1].
 * di_train_grad: forward on the context's current parameters, loss L = scale * sum_b ||x_hat_b - x_b||^2 (
 *                scale = 1/l for the paper's mean over l images) into DEVICE loss[0] (double), and dL/dparams into
 *                DEVICE grads [di_num_params()] (fp32; reductions are deterministic).  y: DEVICE [batch][ldy] fp32,
 *                x_true: DEVICE [batch][n1][n2] fp32.  Phi (the lifting layer) is fixed and not trained.
 *                Data-parallel training all-reduces `grads` across ranks (sum, with scale = 1/global batch) between
 *                di_train_grad and di_sgd_step.
 * di_sgd_step:   vel = momentum * vel + grads; params -= lr * vel; the kernels' weight layouts follow.
 * di_get_params: DEVICE copy of the current parameters.
 * Custom stacks (di_create_args.layers, NEXT-3; per-channel or zero biases, any precision): the same calls with the
 *                parameter vector [W_0 | W_1 | ... | W_L-1 | b_0 | ... | b_L-1] (each W_l [cout][cin][11][11] in the
 *                orientation given to di_create) of di_ctx_num_params(ctx) floats; forward on the context's kernels,
 *                backward on SIMT fp32 weight / data gradient kernels per layer; in TF32 / BF16 contexts di_sgd_step
 *                re-derives the tensor-core weight images on the host and synchronises `stream`.
 * di_ctx_num_params: the length of the context's parameter vector (di_num_params() for the paper's stack), 0 for
 *                contexts that cannot train (full-map biases) or ctx == NULL. */
long long di_num_params(void);
long long di_ctx_num_params(di_ctx ctx);
di_status di_train_grad(di_ctx ctx, const void* y, long long ldy, const float* x_true, int batch, double scale,
                        float* grads, double* loss, void* stream);
di_status di_sgd_step(di_ctx ctx, const float* grads, double lr, double momentum, void* stream);
di_status di_get_params(di_ctx ctx, float* params, void* stream);

/* Destroy a context (NULL -> DI_OK).  Synchronises the device before freeing. */
di_status di_destroy(di_ctx ctx);

const char* di_status_string(di_status s);
const char* di_last_error(void); /* thread-local detail of the last failing call on this thread */

/* Introspection used by tests and the benchmark. */
typedef struct {
  int m, n1, n2, max_batch;
  di_precision precision;
  unsigned flags;
  int launches_per_recover;      /* kernels enqueued by one di_recover                               */
  long long workspace_bytes;     /* device bytes owned by the context                                */
  const char* stage_kernels[4];  /* kernel names of stages 0..3                                      */
} di_info;
di_status di_get_info(di_ctx ctx, di_info* info);

/* Per-stage device timing: when enabled, di_recover records CUDA events around every stage on its own
 * stream; di_stage_times accumulates elapsed milliseconds of stages 0..3 over the calls since the last
 * reset (it synchronises on the last recorded event).  Off by default (no events recorded). */
di_status di_set_profiling(di_ctx ctx, int enable);
di_status di_stage_times(di_ctx ctx, float ms[4], int* calls, int reset);

/* Test hook: run one stage on caller DEVICE buffers in the documented layouts (storage type of the
 * precision, i.e. bf16 for BF16 and fp32 otherwise, except stage 3 output which is fp32):
 *   stage 0: y [batch][m]             -> x_tilde [batch][n1][n2]
 *   stage 1: x_tilde [batch][n1][n2]  -> h1 [batch][n1][n2][64]  (NHWC)
 *   stage 2: h1                       -> h2 [batch][n1][n2][32]  (NHWC)
 *   stage 3: h2                       -> x_hat [batch][n1][n2] fp32 */
di_status di_debug_stage(di_ctx ctx, int stage, const void* in, void* out, int batch, void* stream);

/* Test hook: copy the context's device copy of the lifting matrix's transpose (Phi, or L^T for a learned lifting;
 * storage type, [m][N] row-major) to a host buffer. */
di_status di_debug_get_phi(di_ctx ctx, void* host_out, long long bytes);

#ifdef __cplusplus
}
#endif
#endif /* DEEPINVERSE_H_ */
