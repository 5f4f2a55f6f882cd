// api.cu -- the C ABI of include/deepinverse.h: validation, ownership, weight packing, workspace,
// TMA tensor maps and the launch sequence of x_hat = M(y, Omega).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <array>
#include <new>
#include <vector>

#include "deepinverse.h"
#include "kernels.cuh"

namespace {

thread_local char g_err[512] = "";

// Every entry point switches to the context's device and restores the caller's current device on return.
struct DevGuard {
  int prev = -1;
  bool ok = false;
  explicit DevGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DevGuard(const DevGuard&) = delete;
  DevGuard& operator=(const DevGuard&) = delete;
};

di_status fail(di_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return s;
}

#define CUDA_TRY(x)                                                                                 \
  do {                                                                                              \
    cudaError_t e_ = (x);                                                                           \
    if (e_ != cudaSuccess)                                                                          \
      return fail(e_ == cudaErrorMemoryAllocation ? DI_ERR_OOM : DI_ERR_CUDA, "%s failed: %s (%s:%d)", #x, \
                  cudaGetErrorString(e_), __FILE__, __LINE__);                                      \
  } while (0)

constexpr int K = 11;             // filter size of every layer
constexpr int C1 = 64, C2 = 32;   // filter counts l1, l2 (l3 = 1)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

uint16_t f2bf(float x) {  // round to nearest even (the harness uses the same rule)
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x7FFFFFu)) return 0x7FC0;
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
float bf2f(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float x;
  std::memcpy(&x, &u, 4);
  return x;
}

}  // namespace

struct di_ctx_s {
  int device = 0, num_sms = 0;
  int conv2_balanced = 1;       // conv2 tiles share a unit's outputs evenly (DI_EXP_C2_SPLIT=253 at di_create: 253 + rest)
  int conv2_mixed = 1;          // conv2 mixed 7- / 6-row blocks where they cut the tiles (DI_EXP_C2_MIXED=0 at di_create: off)
  int conv2_cluster = 2;        // conv2 weight-multicast cluster (DI_EXP_NO_MC=1 -> 1, DI_EXP_C2_CLUSTER=4 -> 4 at di_create)
  int m = 0, n1 = 0, n2 = 0, N = 0, max_batch = 0, kpad = 0;
  int pxbn = 256;               // pixel-tile width of the lifting GEMM = row count of a Phi^T block
  di_precision prec = DI_PREC_BF16;
  unsigned flags = 0;
  size_t elt = 2;
  // device buffers
  void* phi = nullptr;          // FP32: Phi [m][N] fp32 ; BF16/TF32: tile-blocked Phi^T (di::phiT_blk_index), storage type
  float* wx1 = nullptr;         // [1][11][11][64]   xcorr orientation, fp32 (bf16-rounded in BF16 mode)
  float* wx2 = nullptr;         // [64][11][11][32]
  float* wx3 = nullptr;         // [32][11][11][1]
  void* wp2 = nullptr;          // conv2 tensor-core weight blocks (BF16 mode)
  void* wp1 = nullptr;          // conv1 tensor-core weight blocks (BF16 mode, SWIZZLE_32B image)
  void* wp3 = nullptr;          // conv3 tensor-core weight blocks (BF16 mode, SWIZZLE_64B image)
  void* wp2t = nullptr;         // conv2 TF32 weight blocks (TF32 mode)
  struct Layer {                // one layer of a custom stack
    int cin = 0, cout = 0;
    float* wx = nullptr;        // FP32: SIMT layout [ci][a][b][co]
    void* wp = nullptr;         // TF32: tensor-core image (conv1 / generic / conv3 layout by position)
    float* b = nullptr;
    CUtensorMap tm;             // TF32: strip map over this layer's input activation
    size_t woff = 0, boff = 0;  // training: offsets of W_l / b_l in params ([W_0 .. W_L-1 | b_0 .. b_L-1])
    float* wt = nullptr;        // training: backward bank [cout][a][b][cin] (rotated, transposed)
    float* keep = nullptr;      // training: this layer's output, fp32 [max_batch][N][cout] (hidden layers)
  };
  std::vector<Layer> stack;     // empty: the paper's three layers (w1..b3)
  float* act[2] = {nullptr, nullptr};   // custom stack: ping-pong activations [max_batch][N][<= 64] fp32
  long long nparams = 0;        // trainable contexts: parameters in `params` (di::N_PARAMS for the paper's stack)
  float* keep_x = nullptr;      // custom-stack training, BF16: x_tilde as fp32
  float *dA = nullptr, *dB = nullptr;   // custom-stack training: ping-pong data gradients [max_batch][N][<= 64] fp32
  float* wpd3 = nullptr;        // training, TF32 mode: layer-3 dgrad bank in the conv1 TF32 layout
  void* wp2db = nullptr;        // training, TF32 mode: layer-2 dgrad bf16 weight blocks (66 x 8 KB)
  CUtensorMap tmDG2s;           // training, TF32 mode: bf16 dG2 strips for the bf16 dgrad2 (box rows R + 10)
  bool has_tmDX = false;
  CUtensorMap tmDX;             // training, TF32 mode: dG3 strips (the conv1 x_tilde map over dxh)
  void *h1b = nullptr, *dg2b = nullptr;   // training, TF32 mode: bf16 copies of h1 / dG2 (layer-2 wgrad operands)
  void* dh1b = nullptr;                   // training, TF32 mode: dH1 in bf16 (bf16 dgrad2 -> wgrad1)
  float* part_w2 = nullptr;     // training, TF32 mode: per-CTA layer-2 wgrad partials
  CUtensorMap tmH1b, tmDG2b;
  CUtensorMap tmH2w;            // training, BF16 mode: bf16 h2 strips for k_wgrad3_tc
  CUtensorMap tmD1w;            // training, TF32/BF16: bf16 dH1 strips for k_wgrad1_tc
  // training (FP32 contexts with per-channel biases): parameters in the API orientation, momentum, backward
  // weight layouts and the backward workspace (allocated on the first di_train_grad)
  float* params = nullptr;      // [W1 | W2 | W3 | b1 | b2 | b3], di::N_PARAMS
  float* vel = nullptr;
  float *wt2 = nullptr, *wt3 = nullptr;
  float *xh_ws = nullptr, *dxh = nullptr, *dh1 = nullptr, *dh2 = nullptr, *part_w = nullptr, *part_b = nullptr;
  double* loss_img = nullptr;
  void* phi_rm = nullptr;       // di_measure: Phi [m][npad] in the storage type (BF16/TF32; built on first use)
  float* phi_sense = nullptr;   // di_measure in FP32 mode when a learned lifting replaced Phi: Phi [m][N]
  void* xs = nullptr;           // di_measure: staged x [max_batch][npad] in the storage type
  int npad = 0;
  float *b1 = nullptr, *b2 = nullptr, *b3 = nullptr;  // per-channel or cropped full maps (nullptr = zero)
  void *xt = nullptr, *h1 = nullptr, *h2 = nullptr, *ystage = nullptr;
  void* yhost_dev = nullptr;    // di_recover_host staging
  size_t yhost_bytes = 0;
  float* xhost_dev = nullptr;
  cudaStream_t cstream = nullptr;               // di_recover_host: device->host copy stream
  cudaEvent_t cev[17] = {};                      // di_recover_host: chunk-done events (+ the y-copy event)
  int host_chunk_ratio = 4;                      // di_recover_host: chunk k+1 = chunk k / ratio (DI_EXP_E2E_RATIO)
  int host_waves = 1;                            // di_recover_host: chunks in whole conv3 waves (DI_EXP_E2E_WAVES=0: off)
  long long ws_bytes = 0;
  CUtensorMap tmPt{}, tmH1{}, tmH2{}, tmX{};
  CUtensorMap tmH1s{};          // BF16, n2 % 64 == 0: conv1's TMA store map over h1 (encode_h1_store)
  CUtensorMap tmPh{};           // BF16, proxy_pair: Phi^T blocks with half-block boxes (k_proxy_pair)
  bool proxy_pair = false;      // the lifting GEMM on CTA pairs (cta_group::2, k_proxy_pair)
  // di_recover_metrics: set for the duration of one call (the bf16 conv3 epilogue fuses the metrics)
  const float* m_xtrue = nullptr;
  double* m_out = nullptr;
  double* mpart = nullptr;      // per-item metric partials of k_conv3_r4 (allocated on first use, max_batch)
  bool fused_metrics = false;   // di_recover_metrics through k_conv3_r4<true> (DI_EXP_FUSED_METRICS=1 at di_create)
  bool has_tmX = false;
  int last_launches = 0;
  bool profiling = false;
  std::vector<std::array<cudaEvent_t, 5>> evpool;  // one set of stage-boundary events per profiled call
  int ev_used = 0;                                  // sets recorded since the last di_stage_times
  float stage_ms[4] = {0, 0, 0, 0};
  int prof_calls = 0;
};

namespace {

di_status encode_2d(CUtensorMap* map, const void* base, bool bf16, int inner, int outer, long long ld_elems,
                    int box_inner, int box_outer) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld_elems * (bf16 ? 2 : 4)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                   const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled (2d) failed: %d", (int)r);
  return DI_OK;
}

// the tile-blocked Phi^T (di::phiT_blk_index) as [blocks][256 rows][kel]: box = one contiguous 32-KB block
// box_rows: tr (k_proxy_tc: one whole block) or tr / 2 (k_proxy_pair: each CTA of a pair loads half of a block)
di_status encode_phiT_blk(CUtensorMap* map, const void* base, bool bf16, long long N, int kpad, int tr,
                          int box_rows = 0) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  const int e = bf16 ? 2 : 4, kel = 128 / e;
  cuuint64_t dims[3] = {(cuuint64_t)kel, (cuuint64_t)tr, (cuuint64_t)((N + tr - 1) / tr) * (cuuint64_t)(kpad / kel)};
  cuuint64_t strides[2] = {128, (cuuint64_t)tr * 128};
  cuuint32_t box[3] = {(cuuint32_t)kel, (cuuint32_t)(box_rows ? box_rows : tr), 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                   const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled (Phi^T blocks) failed: %d", (int)r);
  return DI_OK;
}

di_status encode_h1(CUtensorMap* map, const void* h1, int batch, int n1, int n2, int mixed) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[4] = {64, (cuuint64_t)n2, (cuuint64_t)n1, (cuuint64_t)batch};
  cuuint64_t strides[3] = {64 * 2, (cuuint64_t)n2 * 64 * 2, (cuuint64_t)n1 * n2 * 64 * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)di::conv2_tc_box_cols(n2), (cuuint32_t)di::conv2_tc_box_rows(n1, n2, mixed), 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(h1), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled (h1) failed: %d", (int)r);
  return DI_OK;
}

// conv1's output path (k_conv1_tc): h1 [batch][n1][n2][64] bf16, box = 16 channels (32 B) x 64 columns x 2 rows,
// SWIZZLE_32B -- one epilogue warp's 128 positions x 16 channels, stored by one TMA tensor store
di_status encode_h1_store(CUtensorMap* map, const void* h1, int batch, int n1, int n2) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[4] = {64, (cuuint64_t)n2, (cuuint64_t)n1, (cuuint64_t)batch};
  cuuint64_t strides[3] = {64 * 2, (cuuint64_t)n2 * 64 * 2, (cuuint64_t)n1 * n2 * 64 * 2};
  cuuint32_t box[4] = {16, 64, 2, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(h1), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled (h1 store) failed: %d", (int)r);
  return DI_OK;
}

// h1 [batch][n1][n2][64] fp32 for the TF32 conv2: box = 32 channels (one 128-B swizzle row) x P x 16 rows
di_status encode_h1_f32(CUtensorMap* map, const void* h1, int batch, int n1, int n2) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[4] = {64, (cuuint64_t)n2, (cuuint64_t)n1, (cuuint64_t)batch};
  cuuint64_t strides[3] = {64 * 4, (cuuint64_t)n2 * 64 * 4, (cuuint64_t)n1 * n2 * 64 * 4};
  cuuint32_t box[4] = {32, (cuuint32_t)di::conv_tf32_box_cols(n2), (cuuint32_t)di::conv2_tf32_box_rows(), 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(h1), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled (h1 f32) failed: %d", (int)r);
  return DI_OK;
}

// x_tilde [batch][n1][n2] for the conv1 strip TMA: bf16 (needs n2 % 8 == 0: 16-B row stride) or fp32 for TF32
// (n2 % 4 == 0)
di_status encode_xt(CUtensorMap* map, const void* xt, int batch, int n1, int n2, bool f32 = false) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  const cuuint64_t e = f32 ? 4 : 2;
  cuuint64_t dims[3] = {(cuuint64_t)n2, (cuuint64_t)n1, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)n2 * e, (cuuint64_t)n1 * n2 * e};
  cuuint32_t box[3] = {(cuuint32_t)di::conv1_tc_box_cols(n2),
                       (cuuint32_t)(f32 ? di::conv1_tf32_box_rows() : di::conv1_tc_box_rows()), 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                   const_cast<void*>(xt), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled (x_tilde) failed: %d", (int)r);
  return DI_OK;
}

// h2 [batch][n1][n2][32] for conv3: bf16 (box = all 32 channels = 64 B) or fp32 for TF32 (box = 16 channels = 64 B)
// fp32 NHWC activations with `ch` channels (a multiple of 32) for the TF32 strips of k_conv_tf32 (32-channel box):
// the layer-2 dgrad's dG2 and the interior layers of custom stacks
di_status encode_act_f32(CUtensorMap* map, const void* dg2, int batch, int n1, int n2, int ch) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[4] = {(cuuint64_t)ch, (cuuint64_t)n2, (cuuint64_t)n1, (cuuint64_t)batch};
  cuuint64_t strides[3] = {(cuuint64_t)ch * 4, (cuuint64_t)n2 * ch * 4, (cuuint64_t)n1 * n2 * ch * 4};
  cuuint32_t box[4] = {32, (cuuint32_t)di::conv_tf32_box_cols(n2), (cuuint32_t)di::conv2_tf32_box_rows(), 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(dg2), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled (dG2) failed: %d", (int)r);
  return DI_OK;
}

// bf16 NHWC activations with `ch` channels (64: SWIZZLE_128B, 32: SWIZZLE_64B) for the layer-2 wgrad strips
di_status encode_wg2(CUtensorMap* map, const void* p, int batch, int n1, int n2, int ch, int box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[4] = {(cuuint64_t)ch, (cuuint64_t)n2, (cuuint64_t)n1, (cuuint64_t)batch};
  cuuint64_t strides[3] = {(cuuint64_t)ch * 2, (cuuint64_t)n2 * ch * 2, (cuuint64_t)n1 * n2 * ch * 2};
  cuuint32_t box[4] = {(cuuint32_t)ch, (cuuint32_t)di::wgrad_box_cols(n2), (cuuint32_t)box_rows, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(p), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, ch == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled (wgrad2 operand) failed: %d", (int)r);
  return DI_OK;
}

// bf16 NHWC activation with `pitch` channels per pixel, read `ch` channels at a time (custom BF16 stacks): box
// ch x box_cols x box_rows, SWIZZLE_128B for 64 channels (128-B rows), SWIZZLE_64B for 32
di_status encode_act_bf16(CUtensorMap* map, const void* p, int batch, int n1, int n2, int pitch, int ch, int box_cols,
                          int box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[4] = {(cuuint64_t)pitch, (cuuint64_t)n2, (cuuint64_t)n1, (cuuint64_t)batch};
  cuuint64_t strides[3] = {(cuuint64_t)pitch * 2, (cuuint64_t)n2 * pitch * 2, (cuuint64_t)n1 * n2 * pitch * 2};
  cuuint32_t box[4] = {(cuuint32_t)ch, (cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(p), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, ch == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled (bf16 activation) failed: %d", (int)r);
  return DI_OK;
}

// dG2 [batch][n1][n2][32] bf16 as the strip of the bf16 layer-2 dgrad: box 32 ch x P x (11 + 10) rows, SWIZZLE_64B
di_status encode_dg2b_strip(CUtensorMap* map, const void* p, int batch, int n1, int n2) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[4] = {32, (cuuint64_t)n2, (cuuint64_t)n1, (cuuint64_t)batch};
  cuuint64_t strides[3] = {32 * 2, (cuuint64_t)n2 * 32 * 2, (cuuint64_t)n1 * n2 * 32 * 2};
  cuuint32_t box[4] = {32, (cuuint32_t)di::conv2_tc_box_cols(n2), (cuuint32_t)di::dgrad2_bf16_box_rows(), 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(p), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled (dG2 bf16 strip) failed: %d", (int)r);
  return DI_OK;
}

// bf16 conv3 (k_conv3_r4): [batch][n1][n2][pitch] bf16 (32 channels read) as a 4-D tensor ordered (channel, column,
// IMAGE, row), so that one box of conv3_r4_box_cols(n2) columns x 2 images x conv3_r4_box_rows() rows lands as strip
// rows of [image][column] -- the same image row of an image pair side by side; SWIZZLE_64B (64-B position rows)
di_status encode_h2_pair(CUtensorMap* map, const void* h2, int batch, int n1, int n2, int pitch) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[4] = {(cuuint64_t)pitch, (cuuint64_t)n2, (cuuint64_t)batch, (cuuint64_t)n1};
  cuuint64_t strides[3] = {(cuuint64_t)pitch * 2, (cuuint64_t)n1 * n2 * pitch * 2, (cuuint64_t)n2 * pitch * 2};
  cuuint32_t box[4] = {32, (cuuint32_t)di::conv3_r4_box_cols(n2), 2, (cuuint32_t)di::conv3_r4_box_rows()};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(h2), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled (h2 image pairs) failed: %d", (int)r);
  return DI_OK;
}

di_status encode_h2(CUtensorMap* map, const void* h2, int batch, int n1, int n2, bool f32 = false) {
  if (!f32) return encode_h2_pair(map, h2, batch, n1, n2, 32);
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  const cuuint64_t e = f32 ? 4 : 2;
  cuuint64_t dims[4] = {32, (cuuint64_t)n2, (cuuint64_t)n1, (cuuint64_t)batch};
  cuuint64_t strides[3] = {32 * e, (cuuint64_t)n2 * 32 * e, (cuuint64_t)n1 * n2 * 32 * e};
  cuuint32_t box[4] = {(cuuint32_t)di::conv3_tc_box_ch(f32), (cuuint32_t)di::conv3_tc_box_cols(n2),
                       (cuuint32_t)di::conv3_tc_box_rows(), 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                   const_cast<void*>(h2), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DI_ERR_CUDA, "cuTensorMapEncodeTiled (h2) failed: %d", (int)r);
  return DI_OK;
}

template <typename T>
di_status upload(T** dst, const void* src, size_t bytes, long long* ws) {
  CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(dst), bytes));
  *ws += (long long)bytes;
  if (src) CUDA_TRY(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
  return DI_OK;
}

// xcorr-orientation taps of layer l: wx[co][ci][a][b] = W[co][ci][10-a][10-b] (true convolution, Eq. (1))
// or the taps as given (DI_FLAG_XCORR); optional bf16 rounding.
std::vector<float> xcorr_taps(const float* w, int cout, int cin, bool given_xcorr, bool round_bf16) {
  std::vector<float> out((size_t)cout * cin * K * K);
  for (int co = 0; co < cout; ++co)
    for (int ci = 0; ci < cin; ++ci)
      for (int a = 0; a < K; ++a)
        for (int b = 0; b < K; ++b) {
          const int u = given_xcorr ? a : K - 1 - a, v = given_xcorr ? b : K - 1 - b;
          float x = w[(((size_t)co * cin + ci) * K + u) * K + v];
          if (round_bf16) x = bf2f(f2bf(x));
          out[(((size_t)co * cin + ci) * K + a) * K + b] = x;
        }
  return out;
}

// SIMT layout [ci][a][b][co]
std::vector<float> simt_layout(const std::vector<float>& wx, int cout, int cin) {
  std::vector<float> out(wx.size());
  for (int co = 0; co < cout; ++co)
    for (int ci = 0; ci < cin; ++ci)
      for (int t = 0; t < K * K; ++t) out[((size_t)ci * K * K + t) * cout + co] = wx[((size_t)co * cin + ci) * K * K + t];
  return out;
}

// conv2 tensor-core blocks: block kb = (u = kb/3, v0 = 4*(kb%3)); row = v'*32 + k; 64 ci; SWIZZLE_128B image
std::vector<uint16_t> conv2_tc_pack(const std::vector<float>& wx2) {
  std::vector<uint16_t> out((size_t)di::C2_KBLOCKS * di::C2_KBLOCK_BYTES / 2, 0);
  for (int kb = 0; kb < di::C2_KBLOCKS; ++kb) {
    const int u = kb / 3, v0 = 4 * (kb % 3);
    uint8_t* blk = reinterpret_cast<uint8_t*>(out.data()) + (size_t)kb * di::C2_KBLOCK_BYTES;
    for (int row = 0; row < 128; ++row) {
      const int vp = row / 32, k = row % 32, b = v0 + vp;
      for (int ci = 0; ci < 64; ++ci) {
        const float x = (b < K) ? wx2[(((size_t)k * 64 + ci) * K + u) * K + b] : 0.f;
        const uint16_t h = f2bf(x);
        const size_t off = (size_t)row * 128 + ((((size_t)ci / 8) ^ (row & 7)) << 4) + (ci % 8) * 2;
        std::memcpy(blk + off, &h, 2);
      }
    }
  }
  return out;
}

// TF32 conv2 blocks: K-block kb = h*33 + u*3 + j (channel half h, tap row u, column-tap group v0 = 4j); row
// v'*32 + k, 32 fp32 channels 32h..32h+31 (128 B), SWIZZLE_128B image (16-B chunk = 4 channels).  Values stay fp32:
// the tensor core reads them as TF32.
std::vector<float> conv2_tf32_pack(const std::vector<float>& wx2) {
  std::vector<float> out((size_t)2 * di::C2_KBLOCKS * di::C2_KBLOCK_BYTES / 4, 0.f);
  for (int h = 0; h < 2; ++h)
    for (int kb = 0; kb < di::C2_KBLOCKS; ++kb) {
      const int u = kb / 3, v0 = 4 * (kb % 3);
      uint8_t* blk = reinterpret_cast<uint8_t*>(out.data()) + ((size_t)h * di::C2_KBLOCKS + kb) * di::C2_KBLOCK_BYTES;
      for (int row = 0; row < 128; ++row) {
        const int vp = row / 32, k = row % 32, b = v0 + vp;
        for (int c = 0; c < 32; ++c) {
          const int ci = 32 * h + c;
          const float x = (b < K) ? wx2[(((size_t)k * 64 + ci) * K + u) * K + b] : 0.f;
          const size_t off = (size_t)row * 128 + ((((size_t)c / 4) ^ (row & 7)) << 4) + (c % 4) * 4;
          std::memcpy(blk + off, &x, 4);
        }
      }
    }
  return out;
}

// conv1 tensor-core blocks: block u (2 KB) = 64 filter rows x 16 column taps (v >= 11 zero), bf16, SWIZZLE_32B
// image (16-B chunk h of row m at m*32 + ((h ^ ((m >> 2) & 1)) << 4)).  Row m holds filter m (natural order: the
// epilogue's stmatrix transposes 8-channel blocks, k_conv13_tc.cu).
std::vector<uint16_t> conv1_tc_pack(const std::vector<float>& wx1) {
  std::vector<uint16_t> out(11 * 2048 / 2, 0);
  uint8_t* base = reinterpret_cast<uint8_t*>(out.data());
  for (int u = 0; u < K; ++u)
    for (int m = 0; m < 64; ++m) {
      const int f = m;
      for (int v = 0; v < 16; ++v) {
        const uint16_t h = v < K ? f2bf(wx1[((size_t)f * K + u) * K + v]) : 0;
        const size_t off = (size_t)u * 2048 + m * 32 + ((((size_t)v / 8) ^ ((m >> 2) & 1)) << 4) + (v % 8) * 2;
        std::memcpy(base + off, &h, 2);
      }
    }
  return out;
}


// bf16 conv3, C3R_RP rows stacked in M (k_conv3_r4): the stack T[i] = W[10 - i], i = C3R_IMIN .., zero outside 0..10;
// entry e = i - C3R_IMIN = C3R_ES rows (row v < 11: column tap v) x 32 channels bf16, SWIZZLE_64B -- window k's A
// operand is the 128-row window from T[10 - k]
std::vector<uint16_t> conv3_r4_pack(const std::vector<float>& wx3) {
  const int es = di::C3R_ES;
  std::vector<uint16_t> out((size_t)di::conv3_r4_tpack_bytes() / 2, 0);
  uint8_t* base = reinterpret_cast<uint8_t*>(out.data());
  for (int e = 0; e < di::C3R_NENT; ++e) {
    const int u = 10 - (e + di::C3R_IMIN);
    for (int r = 0; r < es; ++r)
      for (int c = 0; c < 32; ++c) {
        const uint16_t h = (u >= 0 && u < K && r < K) ? f2bf(wx3[((size_t)c * K + u) * K + r]) : 0;
        const size_t rho = (size_t)e * es + r;
        const size_t off = rho * 64 + (((c / 8) ^ ((rho >> 1) & 3)) << 4) + (c % 8) * 2;
        std::memcpy(base + off, &h, 2);
      }
  }
  return out;
}

// TF32 conv1 blocks: block u (4 KB) = 64 filter rows (permuted as in conv1_tc_pack) x 16 fp32 column taps (v >= 11
// zero), SWIZZLE_64B image (16-B chunk j of row m at m*64 + ((j ^ ((m >> 1) & 3)) << 4)).
std::vector<float> conv1_tf32_pack(const std::vector<float>& wx1) {
  std::vector<float> out(11 * 4096 / 4, 0.f);
  uint8_t* base = reinterpret_cast<uint8_t*>(out.data());
  for (int u = 0; u < K; ++u)
    for (int m = 0; m < 64; ++m) {
      const int grp = m / 16, j = m % 16;
      const int f = 16 * grp + (j < 8 ? 2 * j : 2 * (j - 8) + 1);
      for (int v = 0; v < 16; ++v) {
        const float x = v < K ? wx1[((size_t)f * K + u) * K + v] : 0.f;
        const size_t off = (size_t)u * 4096 + m * 64 + ((((size_t)v / 4) ^ ((m >> 1) & 3)) << 4) + (v % 4) * 4;
        std::memcpy(base + off, &x, 4);
      }
    }
  return out;
}

// TF32 conv3 blocks: block (h, u) (2 KB, index h*11 + u) = 32 rows (row v < 11: tap v of tap row u) x 16 fp32
// channels 16h..16h+15, SWIZZLE_64B image (16-B chunk = 4 channels; chunk j of row r at r*64 + ((j ^ ((r>>1)&3)) << 4)).
std::vector<float> conv3_tf32_pack(const std::vector<float>& wx3) {
  std::vector<float> out((size_t)2 * 11 * 2048 / 4, 0.f);
  uint8_t* base = reinterpret_cast<uint8_t*>(out.data());
  for (int h = 0; h < 2; ++h)
    for (int u = 0; u < K; ++u)
      for (int r = 0; r < 32; ++r)
        for (int c = 0; c < 16; ++c) {
          const float x = r < K ? wx3[((size_t)(16 * h + c) * K + u) * K + r] : 0.f;
          const size_t off = (size_t)(h * 11 + u) * 2048 + r * 64 + ((((size_t)c / 4) ^ ((r >> 1) & 3)) << 4) + (c % 4) * 4;
          std::memcpy(base + off, &x, 4);
        }
  return out;
}

// TF32 blocks of a generic C_in -> C_out layer (k_conv_tf32): block (h, u, j), index (h*11 + u)*J + j, J =
// ceil(11 / TAPS), TAPS = 128 / C_out: row v'*C_out + k (tap TAPS j + v', zero past 10), 32 fp32 channels 32h + c,
// SWIZZLE_128B (16-B chunk of 4 channels at row*128 + ((c/4 ^ (row & 7)) << 4)).  conv2_tf32_pack is the
// (64, 32) case.
std::vector<float> conv_tf32_pack(const std::vector<float>& wx, int cin, int cout) {
  const int taps = 128 / cout, J = (K + taps - 1) / taps, nh = cin / 32;
  std::vector<float> out((size_t)nh * K * J * 4096, 0.f);
  uint8_t* base = reinterpret_cast<uint8_t*>(out.data());
  for (int h = 0; h < nh; ++h)
    for (int u = 0; u < K; ++u)
      for (int j = 0; j < J; ++j)
        for (int row = 0; row < 128; ++row) {
          const int v = taps * j + row / cout, k = row % cout;
          for (int c = 0; c < 32; ++c) {
            const float x = v < K ? wx[(((size_t)k * cin + 32 * h + c) * K + u) * K + v] : 0.f;
            const size_t off = (size_t)((h * K + u) * J + j) * 16384 + row * 128 + ((((size_t)c / 4) ^ (row & 7)) << 4) +
                               (c % 4) * 4;
            std::memcpy(base + off, &x, 4);
          }
        }
  return out;
}

// bf16 interior layer of a custom stack on k_conv2_tc<C_in, C_out>: K-block u * J + j (J = ceil(11 / TAPS), TAPS =
// 128 / C_out column taps v0 = TAPS j ..), row v' * C_out + k, C_in channels per row (128 B: SWIZZLE_128B, 64 B:
// SWIZZLE_64B); conv2_tc_pack is the (64, 32) case
std::vector<uint16_t> convg_tc_pack(const std::vector<float>& wx, int cin, int cout) {
  // C_in = 128: two channel halves, K-block h * 11 J + u J + j over channels 64 h .. 64 h + 63 (k_conv2_tc NH = 2)
  const int taps = 128 / cout, J = (K + taps - 1) / taps, nh = cin > 64 ? cin / 64 : 1, cinh = cin / nh;
  const int rb = 2 * cinh;
  const size_t wb = (size_t)128 * rb;
  std::vector<uint16_t> out((size_t)nh * K * J * wb / 2, 0);
  uint8_t* base = reinterpret_cast<uint8_t*>(out.data());
  for (int h = 0; h < nh; ++h)
    for (int u = 0; u < K; ++u)
      for (int j = 0; j < J; ++j)
        for (int row = 0; row < 128; ++row) {
          const int v = taps * j + row / cout, k = row % cout;
          for (int c = 0; c < cinh; ++c) {
            const int ci = h * cinh + c;
            const uint16_t hv = v < K ? f2bf(wx[(((size_t)k * cin + ci) * K + u) * K + v]) : 0;
            const int sw = rb == 128 ? (row & 7) : ((row >> 1) & 3);
            const size_t off = (size_t)((h * K + u) * J + j) * wb + (size_t)row * rb + ((((size_t)c / 8) ^ sw) << 4) +
                               (c % 8) * 2;
            std::memcpy(base + off, &hv, 2);
          }
        }
  return out;
}

// bias: per-channel [cout] or the window of the full map [cout][n1+10][n2+10] that S keeps, as [n1][n2][cout]
// one layer of a custom stack in the layout of the kernel that runs it (di_create, and di_sgd_step's repack in TF32 /
// BF16 contexts): FP32 SIMT [ci][a][b][co]; BF16 k_conv1_tc (64 bank rows) / k_conv2_tc<C_in, C_out> / k_conv3_r4;
// TF32 k_conv1_tf32 / k_conv_tf32<C_in, C_out> / k_conv3_tc.  wx: cross-correlation taps [cout][cin][11][11].
std::vector<uint8_t> pack_stack_layer(di_precision prec, int i, int L, const std::vector<float>& wx, int cin, int cout) {
  auto bytes = [](const auto& v) {
    const uint8_t* p = reinterpret_cast<const uint8_t*>(v.data());
    return std::vector<uint8_t>(p, p + v.size() * sizeof(v[0]));
  };
  if (prec == DI_PREC_FP32) return bytes(simt_layout(wx, cout, cin));
  std::vector<float> w64;
  if (i == 0) {   // the conv1 machinery: 64 bank rows, rows >= cout zero
    w64.assign((size_t)64 * K * K, 0.f);
    std::copy(wx.begin(), wx.end(), w64.begin());
  }
  if (prec == DI_PREC_BF16) {
    if (i == 0) return bytes(conv1_tc_pack(w64));
    if (i == L - 1) return bytes(conv3_r4_pack(wx));
    return bytes(convg_tc_pack(wx, cin, cout));
  }
  if (i == 0) return bytes(conv1_tf32_pack(w64));
  if (i == L - 1) return bytes(conv3_tf32_pack(wx));
  return bytes(conv_tf32_pack(wx, cin, cout));
}

di_status upload_bias(float** dst, const float* b, int cout, bool fullmap, int n1, int n2, long long* ws) {
  *dst = nullptr;
  if (!b) return DI_OK;
  if (!fullmap) return upload(dst, b, (size_t)cout * 4, ws);
  const int h = n1 + K - 1, w = n2 + K - 1, p = (K - 1) / 2;
  std::vector<float> bm((size_t)n1 * n2 * cout);
  for (int r = 0; r < n1; ++r)
    for (int c = 0; c < n2; ++c)
      for (int o = 0; o < cout; ++o) bm[((size_t)r * n2 + c) * cout + o] = b[((size_t)o * h + r + p) * w + c + p];
  return upload(dst, bm.data(), bm.size() * 4, ws);
}

void free_ctx(di_ctx c) {
  if (!c) return;
  for (auto& l : c->stack) {
    if (l.wx) cudaFree(l.wx);
    if (l.wp) cudaFree(l.wp);
    if (l.b) cudaFree(l.b);
    if (l.wt) cudaFree(l.wt);
    if (l.keep) cudaFree(l.keep);
  }
  if (c->keep_x) cudaFree(c->keep_x);
  if (c->dA) cudaFree(c->dA);
  if (c->dB) cudaFree(c->dB);
  for (auto p : c->act)
    if (p) cudaFree(p);
  void* ps[] = {c->mpart, c->phi, c->wx1, c->wx2, c->wx3, c->wp2, c->wp1, c->wp3, c->wp2t, c->wpd3, c->wp2db, c->h1b, c->dg2b, c->dh1b, c->part_w2, c->phi_rm, c->xs, c->params, c->vel,
                c->wt2, c->wt3, c->xh_ws, c->dxh, c->dh1, c->dh2, c->part_w, c->part_b, c->loss_img, c->phi_sense, c->b1, c->b2, c->b3, c->xt, c->h1, c->h2, c->ystage,
                c->yhost_dev, c->xhost_dev};
  for (void* p : ps)
    if (p) cudaFree(p);
  for (auto& set : c->evpool)
    for (auto e : set)
      if (e) cudaEventDestroy(e);
  for (auto e : c->cev)
    if (e) cudaEventDestroy(e);
  if (c->cstream) cudaStreamDestroy(c->cstream);
  delete c;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// stage 0 (lifting) into xt: the path dtype, or fp32 when out_f32 (row-sharded partial proxies)
di_status run_proxy(di_ctx c, const void* y, long long ldy, int batch, void* xt, bool out_f32, cudaStream_t st,
                    int& launches, const di::ProxyScatter* sc = nullptr) {
  const bool bf16 = c->prec == DI_PREC_BF16;
  if (c->prec == DI_PREC_FP32) {
    CUDA_TRY(di::launch_proxy_f32(reinterpret_cast<const float*>(y), ldy, reinterpret_cast<const float*>(c->phi),
                                  c->m, c->N, batch, reinterpret_cast<float*>(xt), st));
    ++launches;
    if (sc) {
      CUDA_TRY(di::launch_scatter_rows(reinterpret_cast<const float*>(xt), batch, c->N, sc, st));
      ++launches;
    }
  } else {
    const void* ysrc = y;
    long long ld = ldy;
    int inner = c->m;
    if (!aligned16(y) || ((size_t)ldy * c->elt) % 16 != 0) {
      CUDA_TRY(di::launch_stage_y(y, ldy, c->m, c->kpad, batch, c->ystage, bf16, st));
      ++launches;
      ysrc = c->ystage, ld = c->kpad, inner = c->kpad;
    }
    CUtensorMap tmY;
    di_status s = encode_2d(&tmY, ysrc, bf16, inner, batch, ld, 128 / (int)c->elt, 128);
    if (s != DI_OK) return s;
    if (c->proxy_pair && bf16 && !out_f32 && !sc)
      CUDA_TRY(di::launch_proxy_pair(&tmY, &c->tmPh, batch, c->N, c->kpad / 64, xt, c->pxbn, st));
    else
      CUDA_TRY(di::launch_proxy_tc(&tmY, &c->tmPt, batch, c->N, c->kpad / (128 / (int)c->elt), xt, !bf16, st,
                                   out_f32, sc, true, c->pxbn));
    ++launches;
  }
  return DI_OK;
}

// custom stack: x_tilde -> layer 0 -> ... -> x_hat, interior activations ping-pong in act[]
// keep (training): every hidden layer's output is also stored as fp32 in layer.keep for the backward
di_status run_stack(di_ctx c, int batch, void* xt, float* xhat, cudaStream_t st, int& launches, bool keep = false) {
  const int L = (int)c->stack.size();
  const int relu_last = (c->flags & DI_FLAG_FINAL_RELU) ? 1 : 0;
  const void* in = xt;
  for (int i = 0; i < L; ++i) {
    const di_ctx_s::Layer& l = c->stack[i];
    float* out = i == L - 1 ? xhat : c->act[i & 1];
    if (c->prec == DI_PREC_TF32) {
      if (i == 0) {
        CUtensorMap tm;
        const CUtensorMap* tmp = &c->tmX;
        if (xt != c->xt || batch != c->max_batch) {
          di_status s = encode_xt(&tm, xt, batch, c->n1, c->n2, true);
          if (s != DI_OK) return s;
          tmp = &tm;
        }
        CUDA_TRY(di::launch_conv1g_tf32(l.cout, tmp, l.wp, l.b, out, batch, c->n1, c->n2, c->num_sms, st));
      } else if (i == L - 1) {
        CUDA_TRY(di::launch_conv3_tc(&l.tm, l.wp, l.b, 0, relu_last, xhat, batch, c->n1, c->n2, c->num_sms, true, st));
      } else {
        CUDA_TRY(di::launch_convg_tf32(l.cin, l.cout, &l.tm, l.wp, l.b, batch, c->n1, c->n2, out, c->num_sms, st));
      }
    } else if (c->prec == DI_PREC_BF16) {   // bf16 activations (act[] holds __nv_bfloat16)
      void* outb = c->act[i & 1];
      if (i == 0) {
        CUtensorMap tm;
        const CUtensorMap* tmp = nullptr;
        if (c->has_tmX) {
          tmp = &c->tmX;
          if (xt != c->xt || batch != c->max_batch) {
            di_status s = encode_xt(&tm, xt, batch, c->n1, c->n2);
            if (s != DI_OK) return s;
            tmp = &tm;
          }
        }
        CUDA_TRY(di::launch_conv1_tc(tmp, nullptr, xt, l.wp, l.b, 0, outb, batch, c->n1, c->n2, c->num_sms, st));
      } else if (i == L - 1) {
        CUDA_TRY(di::launch_conv3_r4(&l.tm, l.wp, l.b, 0, relu_last, xhat, batch, c->n1, c->n2, c->num_sms, st));
      } else {
        CUDA_TRY(di::launch_convg_tc(l.cin, l.cout, &l.tm, l.wp, l.b, batch, c->n1, c->n2, outb, c->num_sms, st));
      }
      ++launches;
      if (keep && i < L - 1)
        CUDA_TRY(di::launch_bf16_to_f32(outb, i == 0 ? 64 : l.cout, l.cout, (size_t)batch * c->N, l.keep, st));
      continue;
    } else {
      if (i == L - 1)
        CUDA_TRY(di::launch_conv3_simt(in, false, l.wx, l.b, 0, relu_last, xhat, batch, c->n1, c->n2, st));
      else
        CUDA_TRY(di::launch_convg_simt(l.cin, l.cout, reinterpret_cast<const float*>(in), l.wx, l.b, out, batch,
                                       c->n1, c->n2, st));
    }
    ++launches;
    if (keep && i < L - 1)
      CUDA_TRY(cudaMemcpyAsync(l.keep, out, (size_t)batch * c->N * l.cout * 4, cudaMemcpyDeviceToDevice, st));
    in = out;
  }
  return DI_OK;
}

// the launch sequence (stages first..last) on caller buffers
di_status run_stages(di_ctx c, int first, int last, const void* y, long long ldy, int batch, void* xt, void* h1,
                     void* h2, float* xhat, cudaStream_t st) {
  const bool bf16 = c->prec == DI_PREC_BF16;
  const int fm = (c->flags & DI_FLAG_FULLMAP_BIAS) ? 1 : 0;
  const int relu3 = (c->flags & DI_FLAG_FINAL_RELU) ? 1 : 0;
  int launches = 0;
  cudaEvent_t* ev = nullptr;
  if (c->profiling) {
    if (c->ev_used == (int)c->evpool.size()) {
      std::array<cudaEvent_t, 5> set{};
      for (auto& e : set) CUDA_TRY(cudaEventCreate(&e));
      c->evpool.push_back(set);
    }
    ev = c->evpool[c->ev_used++].data();
  }
  auto mark = [&](int i) {
    if (ev) cudaEventRecord(ev[i], st);
  };
  mark(first);
  if (first <= 0 && 0 <= last) {
    di_status s0 = run_proxy(c, y, ldy, batch, xt, false, st, launches);
    if (s0 != DI_OK) return s0;
  }
  mark(1);
  if (!c->stack.empty()) {   // custom stack: its layers are one block (stage 1), stages 2 and 3 empty
    if (first <= 1 && 3 <= last) {
      di_status s1 = run_stack(c, batch, xt, xhat, st, launches);
      if (s1 != DI_OK) return s1;
    } else if (last >= 1) {
      return fail(DI_ERR_ARG, "custom stacks run stages 1..3 as one block");
    }
    mark(2), mark(3), mark(4);
    c->last_launches = launches;
    return DI_OK;
  }
  if (first <= 1 && 1 <= last) {
    if (c->prec == DI_PREC_TF32 && c->has_tmX) {
      CUtensorMap tm;
      const CUtensorMap* tmp = &c->tmX;
      if (xt != c->xt || batch != c->max_batch) {
        di_status s = encode_xt(&tm, xt, batch, c->n1, c->n2, true);
        if (s != DI_OK) return s;
        tmp = &tm;
      }
      CUDA_TRY(di::launch_conv1_tf32(tmp, c->wp1, c->b1, fm, reinterpret_cast<float*>(h1), batch, c->n1, c->n2,
                                     c->num_sms, st));
    } else if (bf16) {
      CUtensorMap tm;
      const CUtensorMap* tmp = nullptr;
      if (c->has_tmX) {
        tmp = &c->tmX;
        if (xt != c->xt || batch != c->max_batch) {
          di_status s = encode_xt(&tm, xt, batch, c->n1, c->n2);
          if (s != DI_OK) return s;
          tmp = &tm;
        }
      }
      // h1 leaves by TMA tensor stores when the image rows are whole 64-column segments (k_conv13_tc.cu)
      CUtensorMap ts;
      const CUtensorMap* tsp = nullptr;
      if (c->n2 % 64 == 0) {
        tsp = &c->tmH1s;
        if (h1 != c->h1) {
          di_status s = encode_h1_store(&ts, h1, batch, c->n1, c->n2);
          if (s != DI_OK) return s;
          tsp = &ts;
        }
      }
      CUDA_TRY(di::launch_conv1_tc(tmp, tsp, xt, c->wp1, c->b1, fm, h1, batch, c->n1, c->n2, c->num_sms, st));
    }
    else
      CUDA_TRY(di::launch_conv1_simt(xt, bf16, c->wx1, c->b1, fm, h1, batch, c->n1, c->n2, st));
    ++launches;
  }
  mark(2);
  if (first <= 2 && 2 <= last) {
    if (bf16) {
      CUtensorMap tm;
      const CUtensorMap* tmp = &c->tmH1;
      if (h1 != c->h1 || batch != c->max_batch) {
        di_status s = encode_h1(&tm, h1, batch, c->n1, c->n2, c->conv2_mixed);
        if (s != DI_OK) return s;
        tmp = &tm;
      }
      CUDA_TRY(di::launch_conv2_tc(tmp, c->wp2, c->b2, fm, batch, c->n1, c->n2, h2, c->num_sms, st, c->conv2_cluster,
                                   c->conv2_balanced, c->conv2_mixed));
    } else if (c->prec == DI_PREC_TF32) {
      CUtensorMap tm;
      const CUtensorMap* tmp = &c->tmH1;
      if (h1 != c->h1 || batch != c->max_batch) {
        di_status s = encode_h1_f32(&tm, h1, batch, c->n1, c->n2);
        if (s != DI_OK) return s;
        tmp = &tm;
      }
      CUDA_TRY(di::launch_conv2_tf32(tmp, c->wp2t, c->b2, fm, batch, c->n1, c->n2, reinterpret_cast<float*>(h2),
                                     c->num_sms, st));
    } else {
      CUDA_TRY(di::launch_conv2_simt_f32(reinterpret_cast<const float*>(h1), c->wx2, c->b2, fm,
                                         reinterpret_cast<float*>(h2), batch, c->n1, c->n2, st));
    }
    ++launches;
  }
  mark(3);
  if (first <= 3 && 3 <= last) {
    if (c->prec != DI_PREC_FP32) {
      CUtensorMap tm;
      const CUtensorMap* tmp = &c->tmH2;
      if (h2 != c->h2 || batch != c->max_batch) {
        di_status s = encode_h2(&tm, h2, batch, c->n1, c->n2, !bf16);
        if (s != DI_OK) return s;
        tmp = &tm;
      }
      if (bf16)
        CUDA_TRY(di::launch_conv3_r4(tmp, c->wp3, c->b3, fm, relu3, xhat, batch, c->n1, c->n2, c->num_sms, st,
                                     c->m_xtrue, c->mpart, c->m_out));
      else
        CUDA_TRY(di::launch_conv3_tc(tmp, c->wp3, c->b3, fm, relu3, xhat, batch, c->n1, c->n2, c->num_sms, true, st));
    } else {
      CUDA_TRY(di::launch_conv3_simt(h2, bf16, c->wx3, c->b3, fm, relu3, xhat, batch, c->n1, c->n2, st));
    }
    ++launches;
  }
  mark(4);
  c->last_launches = launches;
  return DI_OK;
}

#ifdef DI_DEBUG
}  // namespace
namespace di {
cudaError_t di_debug_bind_k_proxy(unsigned int*);
cudaError_t di_debug_bind_k_conv13_tc(unsigned int*);
cudaError_t di_debug_bind_k_conv2_tc(unsigned int*);
cudaError_t di_debug_bind_k_conv3_r4(unsigned int*);
cudaError_t di_debug_bind_k_conv2_tf32(unsigned int*);
cudaError_t di_debug_bind_k_wgrad13_tc(unsigned int*);
cudaError_t di_debug_bind_k_wgrad2_tc(unsigned int*);
}  // namespace di
namespace {
// one host-mapped record per process, bound into every kernel translation unit of the current device
volatile unsigned int* debug_record() {
  static unsigned int* host = nullptr;
  if (!host) {
    if (cudaHostAlloc(reinterpret_cast<void**>(&host), 64, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
      return nullptr;
    std::memset(host, 0, 64);
  }
  return host;
}
di_status debug_bind() {
  volatile unsigned int* h = debug_record();
  if (!h) return fail(DI_ERR_CUDA, "debug record allocation failed");
  unsigned int* d = nullptr;
  CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d), const_cast<unsigned int*>(h), 0));
  CUDA_TRY(di::di_debug_bind_k_proxy(d));
  CUDA_TRY(di::di_debug_bind_k_conv13_tc(d));
  CUDA_TRY(di::di_debug_bind_k_conv2_tc(d));
  CUDA_TRY(di::di_debug_bind_k_conv3_r4(d));
  CUDA_TRY(di::di_debug_bind_k_conv2_tf32(d));
  CUDA_TRY(di::di_debug_bind_k_wgrad13_tc(d));
  CUDA_TRY(di::di_debug_bind_k_wgrad2_tc(d));
  return DI_OK;
}
#endif

}  // namespace

extern "C" {

#ifdef DI_EXPERIMENT_BUILD
// present only in libdeepinverse_exp.so (tests/test_abi.py asserts the product library does not export it)
__attribute__((visibility("default"))) extern const char di_experiment_build[] = "experiment build";
#endif

#ifdef DI_DEBUG
// Debug library only (sm100.cuh DI_DEBUG): the host-mapped failure record of bounded mbarrier waits and device
// asserts.  Returns the record's code (0 = no failure) and formats it into buf.
static const char* const kTuNames[] = {"?", "k_proxy", "k_conv13_tc", "k_conv2_tc", "k_conv3_r4", "k_conv2_tf32",
                                       "k_sense", "k_train", "k_wgrad13_tc", "k_wgrad2_tc", "k_conv_simt"};
int di_debug_report(char* buf, int n) {
  volatile unsigned int* r = debug_record();
  if (!r) return -1;
  const unsigned int code = r[0];
  if (buf && n > 0) {
    const unsigned int tu = code >> 8, kind = code & 0xff;
    snprintf(buf, n, "%s: %s in %s, block %u thread %u (a=0x%x b=%u)", code ? "FAILED" : "ok",
             kind == 1 ? "mbarrier wait timed out" : kind == 2 ? "device assert" : "-",
             tu < sizeof(kTuNames) / sizeof(kTuNames[0]) ? kTuNames[tu] : "?", r[1], r[2], r[3], r[4]);
  }
  return (int)code;
}
#endif

const char* di_status_string(di_status s) {
  switch (s) {
    case DI_OK: return "DI_OK";
    case DI_ERR_ARG: return "DI_ERR_ARG";
    case DI_ERR_DIM: return "DI_ERR_DIM";
    case DI_ERR_DOMAIN: return "DI_ERR_DOMAIN";
    case DI_ERR_DEVICE: return "DI_ERR_DEVICE";
    case DI_ERR_OOM: return "DI_ERR_OOM";
    case DI_ERR_CUDA: return "DI_ERR_CUDA";
  }
  return "DI_ERR_UNKNOWN";
}

const char* di_last_error(void) { return g_err; }

di_status di_create(const di_create_args* a, di_ctx* out) {
  if (!out) return fail(DI_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (!a) return fail(DI_ERR_ARG, "args is NULL");
  if (a->n1 < 1 || a->n2 < 1) return fail(DI_ERR_DOMAIN, "n1=%d n2=%d must be >= 1", a->n1, a->n2);
  const long long N = (long long)a->n1 * a->n2;
  if (a->m < 1 || a->m > N) return fail(DI_ERR_DOMAIN, "m=%d must satisfy 1 <= m <= N=%lld (SPEC.md:140)", a->m, N);
  const bool custom = a->n_layers != 0;
  if (!a->phi) return fail(DI_ERR_ARG, "phi must be non-NULL");
  if (!custom && (!a->w1 || !a->w2 || !a->w3)) return fail(DI_ERR_ARG, "w1..w3 must be non-NULL");
  if (custom) {   // SURVEY.md §8(f) NEXT-3 custom stacks: shapes the kernels implement
    const int L = a->n_layers;
    if (L < 2 || !a->layers) return fail(DI_ERR_ARG, "n_layers=%d: a custom stack needs >= 2 layers", L);
    if (a->flags & DI_FLAG_FULLMAP_BIAS) return fail(DI_ERR_ARG, "custom stacks take per-channel biases");
    if (a->precision == DI_PREC_TF32 && a->n2 % 4 != 0) return fail(DI_ERR_ARG, "TF32 custom stacks need n2 %% 4 == 0");
    for (int i = 0; i < L; ++i) {
      const di_layer& l = a->layers[i];
      if (!l.w) return fail(DI_ERR_ARG, "layers[%d].w is NULL", i);
      if (i > 0 && l.cin != a->layers[i - 1].cout)
        return fail(DI_ERR_DIM, "layers[%d].cin=%d != layers[%d].cout=%d", i, l.cin, i - 1, a->layers[i - 1].cout);
      const bool w32_64 = (l.cout == 32 || l.cout == 64);
      auto wide = [](int c) { return c == 32 || c == 64 || c == 128; };
      const bool ok = i == 0 ? (l.cin == 1 && w32_64) : i == L - 1 ? (l.cin == 32 && l.cout == 1)
                                                                   : (wide(l.cin) && wide(l.cout));
      if (!ok)
        return fail(DI_ERR_ARG, "layers[%d] %d -> %d unsupported (first 1 -> {32,64}, interior {32,64,128} -> "
                    "{32,64,128}, last 32 -> 1)", i, l.cin, l.cout);
      if (a->precision == DI_PREC_TF32 && (l.cin == 128 || l.cout == 128))
        return fail(DI_ERR_ARG, "layers[%d]: width 128 runs in FP32 and BF16 contexts (the TF32 interior kernel "
                    "keeps C_in fp32 channels of the strip in shared memory)", i);
    }
  }
  if (a->phi_dtype != DI_DTYPE_F32 && a->phi_dtype != DI_DTYPE_BF16) return fail(DI_ERR_ARG, "bad phi_dtype");
  if (a->precision != DI_PREC_FP32 && a->precision != DI_PREC_TF32 && a->precision != DI_PREC_BF16)
    return fail(DI_ERR_ARG, "bad precision %d", (int)a->precision);
  if (a->flags & ~(unsigned)(DI_FLAG_XCORR | DI_FLAG_FULLMAP_BIAS | DI_FLAG_FINAL_RELU))
    return fail(DI_ERR_ARG, "unknown flag bits 0x%x", a->flags);
  if (a->max_batch < 1) return fail(DI_ERR_ARG, "max_batch=%d must be >= 1", a->max_batch);
  if (a->precision != DI_PREC_FP32 && N > 0x7fffffffLL) return fail(DI_ERR_DIM, "N too large");

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(DI_ERR_DEVICE, "no CUDA device");
  if (a->device < 0 || a->device >= ndev) return fail(DI_ERR_DEVICE, "device %d out of range", a->device);
  int maj = 0, min = 0;
  cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, a->device);
  cudaDeviceGetAttribute(&min, cudaDevAttrComputeCapabilityMinor, a->device);
  if (maj != 10 || min != 0)
    return fail(DI_ERR_DEVICE, "device %d is sm_%d%d; this library is built for sm_100a only", a->device, maj, min);
  DevGuard dg_(a->device);
  if (!dg_.ok) return fail(DI_ERR_CUDA, "cudaSetDevice(%d) failed", a->device);

  di_ctx c = new (std::nothrow) di_ctx_s();
  if (!c) return fail(DI_ERR_OOM, "host allocation failed");
  c->device = a->device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, a->device);
  // read once per context, never on the launch path (A/B switches of the multicast cluster)
  c->conv2_cluster = getenv("DI_EXP_NO_MC") ? 1 : (getenv("DI_EXP_C2_CLUSTER") ? atoi(getenv("DI_EXP_C2_CLUSTER")) : 2);
  c->fused_metrics = getenv("DI_EXP_FUSED_METRICS") != nullptr && atoi(getenv("DI_EXP_FUSED_METRICS")) != 0;
  c->conv2_balanced = !(getenv("DI_EXP_C2_SPLIT") && atoi(getenv("DI_EXP_C2_SPLIT")) == 253);
  c->conv2_mixed = !(getenv("DI_EXP_C2_MIXED") && atoi(getenv("DI_EXP_C2_MIXED")) == 0);
  c->host_chunk_ratio = getenv("DI_EXP_E2E_RATIO") ? std::max(2, atoi(getenv("DI_EXP_E2E_RATIO"))) : 4;
  c->host_waves = !(getenv("DI_EXP_E2E_WAVES") && atoi(getenv("DI_EXP_E2E_WAVES")) == 0);
#ifdef DI_DEBUG
  {
    di_status sd = debug_bind();
    if (sd != DI_OK) {
      delete c;
      return sd;
    }
  }
#endif
  c->m = a->m, c->n1 = a->n1, c->n2 = a->n2, c->N = (int)N, c->max_batch = a->max_batch;
  c->prec = a->precision, c->flags = a->flags;
  c->elt = (a->precision == DI_PREC_BF16) ? 2 : 4;
  c->kpad = ((a->m + 63) / 64) * 64;
  const bool bf16 = c->prec == DI_PREC_BF16;
  const bool xc = (a->flags & DI_FLAG_XCORR) != 0, fm = (a->flags & DI_FLAG_FULLMAP_BIAS) != 0;
  di_status s = DI_OK;
#define STEP(x)              \
  do {                       \
    s = (x);                 \
    if (s != DI_OK) {        \
      free_ctx(c);           \
      return s;              \
    }                        \
  } while (0)

  // ---- the lifting matrix (Phi^T, or a learned L) as its transpose [m][N]: upload as fp32, then pack on the device
  std::vector<float> phif;   // Phi as fp32 (kept for di_measure when a learned lifting replaces Phi^T)
  const float* phi32 = reinterpret_cast<const float*>(a->phi);
  if (a->phi_dtype == DI_DTYPE_BF16) {
    phif.resize((size_t)a->m * N);
    const uint16_t* pb = reinterpret_cast<const uint16_t*>(a->phi);
    for (size_t i = 0; i < phif.size(); ++i) phif[i] = bf2f(pb[i]);
    phi32 = phif.data();
  }
  {
    std::vector<float> liftT;
    const float* phisrc = phi32;
    if (a->lift) {                                  // L [N][m] -> L^T [m][N]
      liftT.resize((size_t)a->m * N);
      for (long long j = 0; j < N; ++j)
        for (int i = 0; i < a->m; ++i) liftT[(size_t)i * N + j] = a->lift[(size_t)j * a->m + i];
      phisrc = liftT.data();
    }
    if (c->prec == DI_PREC_FP32) {
      STEP(upload(reinterpret_cast<float**>(&c->phi), phisrc, (size_t)a->m * N * 4, &c->ws_bytes));
    } else {
      float* tmp = nullptr;
      long long dummy = 0;
      STEP(upload(&tmp, phisrc, (size_t)a->m * N * 4, &dummy));
      c->pxbn = di::proxy_tile_width(N, a->max_batch, bf16, c->num_sms);
      // CTA pairs when Phi is large enough to stream from HBM (N >= 16384: Larger, Stress) and the batch fills the
      // 256-image pair tile; DI_EXP_PROXY_PAIR=0/1 at di_create overrides (A/B runs)
      c->proxy_pair = bf16 && N >= 16384 && a->max_batch >= 256;
      if (const char* ev = getenv("DI_EXP_PROXY_PAIR")) c->proxy_pair = bf16 && atoi(ev) != 0;
      const size_t bytes = di::phiT_blk_elems(N, c->kpad, c->pxbn) * c->elt;   // tile-blocked, zero rows past N
      cudaError_t e = cudaMalloc(&c->phi, bytes);
      if (e == cudaSuccess) e = cudaMemset(c->phi, 0, bytes);
      if (e != cudaSuccess) {
        cudaFree(tmp);
        free_ctx(c);
        return fail(DI_ERR_OOM, "cudaMalloc(Phi^T, %zu) failed", bytes);
      }
      c->ws_bytes += bytes;
      e = di::launch_pack_phiT(tmp, a->m, (int)N, c->kpad, c->pxbn, c->phi, bf16, 0);
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      cudaFree(tmp);
      if (e != cudaSuccess) {
        free_ctx(c);
        return fail(DI_ERR_CUDA, "packing Phi^T failed: %s", cudaGetErrorString(e));
      }
    }
  }
  // ---- a learned lifting replaces Phi^T in the proxy only; di_measure keeps sensing with Phi
  if (a->lift) {
    if (c->prec == DI_PREC_FP32) {
      STEP(upload(&c->phi_sense, phi32, (size_t)a->m * N * 4, &c->ws_bytes));
    } else {
      const int kel = 128 / (int)c->elt;
      c->npad = (int)(((N + kel - 1) / kel) * kel);
      std::vector<uint8_t> prm((size_t)a->m * c->npad * c->elt, 0);
      for (int i = 0; i < a->m; ++i)
        for (long long j = 0; j < N; ++j) {
          const float v = phi32[(size_t)i * N + j];
          uint8_t* d = prm.data() + ((size_t)i * c->npad + j) * c->elt;
          if (bf16) {
            const uint16_t h = f2bf(v);
            std::memcpy(d, &h, 2);
          } else {
            std::memcpy(d, &v, 4);
          }
        }
      STEP(upload(reinterpret_cast<uint8_t**>(&c->phi_rm), prm.data(), prm.size(), &c->ws_bytes));
      STEP(upload(reinterpret_cast<uint8_t**>(&c->xs), nullptr, (size_t)a->max_batch * c->npad * c->elt, &c->ws_bytes));
    }
  }
  // ---- weights / biases
  if (custom) {   // the custom stack's banks in the layout of the kernel that runs each layer
    const int L = a->n_layers;
    c->stack.resize(L);
    for (int i = 0; i < L; ++i) {
      const di_layer& al = a->layers[i];
      di_ctx_s::Layer& l = c->stack[i];
      l.cin = al.cin, l.cout = al.cout;
      auto wx = xcorr_taps(al.w, al.cout, al.cin, xc, false);
      const std::vector<uint8_t> img = pack_stack_layer(c->prec, i, L, wx, al.cin, al.cout);
      if (c->prec == DI_PREC_FP32)
        STEP(upload(&l.wx, img.data(), img.size(), &c->ws_bytes));
      else
        STEP(upload(reinterpret_cast<uint8_t**>(&l.wp), img.data(), img.size(), &c->ws_bytes));
      if (bf16 && i == 0 && al.cout < 64 && al.b) {   // k_conv1_tc reads 64 biases: zero past cout
        std::vector<float> b64(64, 0.f);
        std::copy(al.b, al.b + al.cout, b64.begin());
        STEP(upload_bias(&l.b, b64.data(), 64, false, a->n1, a->n2, &c->ws_bytes));
      } else {
        STEP(upload_bias(&l.b, al.b, al.cout, false, a->n1, a->n2, &c->ws_bytes));
      }
    }
    // trainable (NEXT-3): fp32 master parameters [W_0 .. W_L-1 | b_0 .. b_L-1] in the API orientation
    size_t nw = 0, nb = 0;
    for (auto& l : c->stack) l.woff = nw, nw += (size_t)l.cout * l.cin * K * K;
    for (auto& l : c->stack) l.boff = nb, nb += (size_t)l.cout;
    std::vector<float> prm(nw + nb, 0.f);
    for (int i = 0; i < L; ++i) {
      const di_layer& al = a->layers[i];
      const di_ctx_s::Layer& l = c->stack[i];
      std::memcpy(prm.data() + l.woff, al.w, (size_t)l.cout * l.cin * K * K * 4);
      if (al.b) std::memcpy(prm.data() + nw + l.boff, al.b, (size_t)l.cout * 4);
    }
    c->nparams = (long long)prm.size();
    STEP(upload(&c->params, prm.data(), prm.size() * 4, &c->ws_bytes));
    STEP(upload(&c->vel, nullptr, prm.size() * 4, &c->ws_bytes));
    CUDA_TRY(cudaMemset(c->vel, 0, prm.size() * 4));
  } else {
    auto w1 = xcorr_taps(a->w1, C1, 1, xc, bf16);
    auto w2 = xcorr_taps(a->w2, C2, C1, xc, bf16);
    auto w3 = xcorr_taps(a->w3, 1, C2, xc, bf16);
    auto s1 = simt_layout(w1, C1, 1), s2 = simt_layout(w2, C2, C1), s3 = simt_layout(w3, 1, C2);
    STEP(upload(&c->wx1, s1.data(), s1.size() * 4, &c->ws_bytes));
    STEP(upload(&c->wx2, s2.data(), s2.size() * 4, &c->ws_bytes));
    STEP(upload(&c->wx3, s3.data(), s3.size() * 4, &c->ws_bytes));
    if (bf16) {
      auto p2 = conv2_tc_pack(w2);
      STEP(upload(&c->wp2, p2.data(), p2.size() * 2, &c->ws_bytes));
      auto p1 = conv1_tc_pack(w1);
      STEP(upload(&c->wp1, p1.data(), p1.size() * 2, &c->ws_bytes));
      auto p3 = conv3_r4_pack(w3);
      STEP(upload(&c->wp3, p3.data(), p3.size() * 2, &c->ws_bytes));
    }
    if (c->prec == DI_PREC_TF32) {
      auto pt = conv2_tf32_pack(w2);
      STEP(upload(&c->wp2t, pt.data(), pt.size() * 4, &c->ws_bytes));
      auto p3 = conv3_tf32_pack(w3);
      STEP(upload(&c->wp3, p3.data(), p3.size() * 4, &c->ws_bytes));
      auto p1 = conv1_tf32_pack(w1);
      STEP(upload(&c->wp1, p1.data(), p1.size() * 4, &c->ws_bytes));
    }
    STEP(upload_bias(&c->b1, a->b1, C1, fm, a->n1, a->n2, &c->ws_bytes));
    STEP(upload_bias(&c->b2, a->b2, C2, fm, a->n1, a->n2, &c->ws_bytes));
    STEP(upload_bias(&c->b3, a->b3, 1, fm, a->n1, a->n2, &c->ws_bytes));
    if (!fm) {   // trainable: fp32 master parameters in the API orientation
      c->nparams = di::N_PARAMS;
      std::vector<float> prm(di::N_PARAMS, 0.f);
      const size_t n1w = (size_t)C1 * K * K, n2w = (size_t)C2 * C1 * K * K, n3w = (size_t)C2 * K * K;
      std::memcpy(prm.data(), a->w1, n1w * 4);
      std::memcpy(prm.data() + n1w, a->w2, n2w * 4);
      std::memcpy(prm.data() + n1w + n2w, a->w3, n3w * 4);
      float* pb = prm.data() + n1w + n2w + n3w;
      if (a->b1) std::memcpy(pb, a->b1, C1 * 4);
      if (a->b2) std::memcpy(pb + C1, a->b2, C2 * 4);
      if (a->b3) std::memcpy(pb + C1 + C2, a->b3, 4);
      STEP(upload(&c->params, prm.data(), prm.size() * 4, &c->ws_bytes));
      STEP(upload(&c->vel, nullptr, prm.size() * 4, &c->ws_bytes));
      CUDA_TRY(cudaMemset(c->vel, 0, prm.size() * 4));
    }
  }
  // ---- workspace
  {
    const size_t B = (size_t)a->max_batch;
    STEP(upload(&c->xt, nullptr, B * N * c->elt, &c->ws_bytes));
    if (custom) {
      int wmax = 0;
      for (const auto& l : c->stack) wmax = std::max(wmax, l.cout);
      // BF16: bf16 activations, the first layer's at pitch 64 (k_conv1_tc writes 64 channels, the rows >= cout zero)
      if (bf16) wmax = std::max(wmax, 64);
      for (auto& p : c->act) STEP(upload(&p, nullptr, B * N * wmax * (bf16 ? 2 : 4), &c->ws_bytes));
    } else {
      STEP(upload(&c->h1, nullptr, B * N * C1 * c->elt, &c->ws_bytes));
      STEP(upload(&c->h2, nullptr, B * N * C2 * c->elt, &c->ws_bytes));
    }
    if (c->prec != DI_PREC_FP32) STEP(upload(&c->ystage, nullptr, B * c->kpad * c->elt, &c->ws_bytes));
  }
  // ---- kernels / tensor maps
  if (c->prec == DI_PREC_TF32) {
    cudaError_t e = di::setup_conv2_tf32(a->n2);
    if (e != cudaSuccess) {
      free_ctx(c);
      return fail(DI_ERR_CUDA, "setup_conv2_tf32: %s", cudaGetErrorString(e));
    }
    e = di::setup_conv13_tc(a->n2);
    if (e != cudaSuccess) {
      free_ctx(c);
      return fail(DI_ERR_CUDA, "setup_conv13_tc: %s", cudaGetErrorString(e));
    }
    if (custom) {   // each layer's input strip map over the ping-pong buffer it reads
      for (int i = 1; i < (int)c->stack.size(); ++i) {
        di_ctx_s::Layer& l = c->stack[i];
        if (i == (int)c->stack.size() - 1)
          STEP(encode_h2(&l.tm, c->act[(i - 1) & 1], a->max_batch, a->n1, a->n2, true));
        else
          STEP(encode_act_f32(&l.tm, c->act[(i - 1) & 1], a->max_batch, a->n1, a->n2, l.cin));
      }
    } else {
      STEP(encode_h1_f32(&c->tmH1, c->h1, a->max_batch, a->n1, a->n2));
      STEP(encode_h2(&c->tmH2, c->h2, a->max_batch, a->n1, a->n2, true));
    }
    if (a->n2 % 4 == 0) {
      STEP(encode_xt(&c->tmX, c->xt, a->max_batch, a->n1, a->n2, true));
      c->has_tmX = true;
    }
  }
  if (c->prec != DI_PREC_FP32) {
    cudaError_t e = di::setup_proxy_tc();
    if (e == cudaSuccess) e = di::setup_proxy_pair();
    if (e != cudaSuccess) {
      free_ctx(c);
      return fail(DI_ERR_CUDA, "setup_proxy_tc: %s", cudaGetErrorString(e));
    }
    STEP(encode_phiT_blk(&c->tmPt, c->phi, bf16, N, c->kpad, c->pxbn));
    if (c->proxy_pair) STEP(encode_phiT_blk(&c->tmPh, c->phi, bf16, N, c->kpad, c->pxbn, c->pxbn / 2));
  }
  if (bf16) {
    cudaError_t e = di::setup_conv2_tc(a->n2);
    if (e == cudaSuccess && custom) e = di::setup_convg_tc(a->n2);
    if (e != cudaSuccess) {
      free_ctx(c);
      return fail(DI_ERR_CUDA, "setup_conv2_tc: %s", cudaGetErrorString(e));
    }
    if (custom) {   // layer i >= 1 reads act[(i - 1) & 1] (pitch 64 after the first layer, else the previous C_out)
      for (int i = 1; i < (int)c->stack.size(); ++i) {
        di_ctx_s::Layer& l = c->stack[i];
        const int pitch = i == 1 ? 64 : c->stack[i - 1].cout;
        const bool last = i == (int)c->stack.size() - 1;
        if (last)
          STEP(encode_h2_pair(&l.tm, c->act[(i - 1) & 1], a->max_batch, a->n1, a->n2, pitch));
        else
          STEP(encode_act_bf16(&l.tm, c->act[(i - 1) & 1], a->max_batch, a->n1, a->n2, pitch, std::min(l.cin, 64),
                               di::conv2_tc_box_cols(a->n2), di::convg_tc_box_rows(l.cin)));
      }
    } else {
      STEP(encode_h1(&c->tmH1, c->h1, a->max_batch, a->n1, a->n2, c->conv2_mixed));
      if (a->n2 % 64 == 0) STEP(encode_h1_store(&c->tmH1s, c->h1, a->max_batch, a->n1, a->n2));
    }
    e = di::setup_conv13_tc(a->n2);
    if (e != cudaSuccess) {
      free_ctx(c);
      return fail(DI_ERR_CUDA, "setup_conv13_tc: %s", cudaGetErrorString(e));
    }
    if (!custom) STEP(encode_h2(&c->tmH2, c->h2, a->max_batch, a->n1, a->n2));
    {
      cudaError_t e3 = di::setup_conv3_r4(a->n2);
      if (e3 != cudaSuccess) {
        free_ctx(c);
        return fail(DI_ERR_CUDA, "setup_conv3_r4: %s", cudaGetErrorString(e3));
      }
    }
    if (a->n2 % 8 == 0) {
      STEP(encode_xt(&c->tmX, c->xt, a->max_batch, a->n1, a->n2));
      c->has_tmX = true;
    }
  }
#undef STEP
  *out = c;
  return DI_OK;
}

di_status di_recover(di_ctx c, const void* y, long long ldy, int batch, float* xhat, void* stream) {
  if (!c) return fail(DI_ERR_ARG, "ctx is NULL");
  if (!y || !xhat) return fail(DI_ERR_ARG, "y and xhat must be non-NULL device pointers");
  if (batch < 1 || batch > c->max_batch) return fail(DI_ERR_ARG, "batch=%d outside [1, %d]", batch, c->max_batch);
  if (ldy < c->m) return fail(DI_ERR_DIM, "ldy=%lld < m=%d", ldy, c->m);
  DevGuard dg_(c->device);
  if (!dg_.ok) return fail(DI_ERR_CUDA, "cudaSetDevice(%d) failed", c->device);
  return run_stages(c, 0, 3, y, ldy, batch, c->xt, c->h1, c->h2, xhat, reinterpret_cast<cudaStream_t>(stream));
}

di_status di_recover_metrics(di_ctx c, const void* y, long long ldy, int batch, const float* x_true, float* xhat,
                             double* metrics, void* stream) {
  if (!c) return fail(DI_ERR_ARG, "ctx is NULL");
  if (!y || !xhat || !x_true || !metrics) return fail(DI_ERR_ARG, "y, x_true, xhat and metrics must be non-NULL");
  if (batch < 1 || batch > c->max_batch) return fail(DI_ERR_ARG, "batch=%d outside [1, %d]", batch, c->max_batch);
  if (ldy < c->m) return fail(DI_ERR_DIM, "ldy=%lld < m=%d", ldy, c->m);
  DevGuard dg_(c->device);
  if (!dg_.ok) return fail(DI_ERR_CUDA, "cudaSetDevice(%d) failed", c->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // The fused epilogue (k_conv3_r4<true>) measured slower than recover + the separate k_metrics pass (7.64 vs 7.60 ms
  // per 4096 64x64 images: the fp64 sums lengthen conv3's epilogue, which is on its critical path), so it runs only
  // when the context was created with DI_EXP_FUSED_METRICS=1 (A/B)
  const bool fused = c->fused_metrics && c->prec == DI_PREC_BF16 && c->stack.empty();
  if (fused) {
    if (!c->mpart)
      CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&c->mpart),
                          di::conv3_r4_metrics_part_bytes(c->max_batch, c->n1, c->n2, c->num_sms)));
    c->m_xtrue = x_true, c->m_out = metrics;
  }
  di_status s = run_stages(c, 0, 3, y, ldy, batch, c->xt, c->h1, c->h2, xhat, st);
  c->m_xtrue = nullptr, c->m_out = nullptr;
  if (s != DI_OK || fused) return s;
  CUDA_TRY(di::launch_metrics(xhat, x_true, c->N, batch, metrics, st));   // other paths: the separate pass
  return DI_OK;
}

di_status di_proxy_partial(di_ctx c, const void* y, long long ldy, int batch, float* xt_part, void* stream) {
  if (!c) return fail(DI_ERR_ARG, "ctx is NULL");
  if (!y || !xt_part) return fail(DI_ERR_ARG, "y and xt_part must be non-NULL device pointers");
  if (batch < 1 || batch > c->max_batch) return fail(DI_ERR_ARG, "batch=%d outside [1, %d]", batch, c->max_batch);
  if (ldy < c->m) return fail(DI_ERR_DIM, "ldy=%lld < m=%d", ldy, c->m);
  DevGuard dg_(c->device);
  if (!dg_.ok) return fail(DI_ERR_CUDA, "cudaSetDevice(%d) failed", c->device);
  int launches = 0;
  return run_proxy(c, y, ldy, batch, xt_part, true, reinterpret_cast<cudaStream_t>(stream), launches);
}

di_status di_proxy_scatter(di_ctx c, const void* y, long long ldy, int batch, float* const* slots, int world, int rank,
                           void* stream) {
  if (!c) return fail(DI_ERR_ARG, "ctx is NULL");
  if (!y || !slots) return fail(DI_ERR_ARG, "y and slots must be non-NULL");
  if (world < 1 || world > 8 || rank < 0 || rank >= world)
    return fail(DI_ERR_ARG, "world=%d rank=%d: need 1 <= world <= 8, 0 <= rank < world", world, rank);
  if (batch < 1 || batch > c->max_batch || batch % world != 0)
    return fail(DI_ERR_ARG, "batch=%d must be in [1, %d] and a multiple of world=%d", batch, c->max_batch, world);
  if (ldy < c->m) return fail(DI_ERR_DIM, "ldy=%lld < m=%d", ldy, c->m);
  di::ProxyScatter sc{};
  for (int r = 0; r < world; ++r) {
    if (!slots[r]) return fail(DI_ERR_ARG, "slots[%d] is NULL", r);
    sc.slots[r] = slots[r];
  }
  sc.world = world, sc.rank = rank, sc.nb = batch / world;
  DevGuard dg_(c->device);
  if (!dg_.ok) return fail(DI_ERR_CUDA, "cudaSetDevice(%d) failed", c->device);
  int launches = 0;
  return run_proxy(c, y, ldy, batch, c->xt, true, reinterpret_cast<cudaStream_t>(stream), launches, &sc);
}

di_status di_recover_from_slots(di_ctx c, const float* staging, int world, int nb, float* xhat, void* stream) {
  if (!c) return fail(DI_ERR_ARG, "ctx is NULL");
  if (!staging || !xhat) return fail(DI_ERR_ARG, "staging and xhat must be non-NULL device pointers");
  if (world < 1 || world > 8) return fail(DI_ERR_ARG, "world=%d outside [1, 8]", world);
  if (nb < 1 || nb > c->max_batch) return fail(DI_ERR_ARG, "nb=%d outside [1, %d]", nb, c->max_batch);
  DevGuard dg_(c->device);
  if (!dg_.ok) return fail(DI_ERR_CUDA, "cudaSetDevice(%d) failed", c->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  CUDA_TRY(di::launch_reduce_slots(staging, world, nb, c->N, c->xt, c->prec == DI_PREC_BF16, st));
  return run_stages(c, 1, 3, nullptr, 0, nb, c->xt, c->h1, c->h2, xhat, st);
}

di_status di_recover_from_proxy(di_ctx c, const float* xt, int batch, float* xhat, void* stream) {
  if (!c) return fail(DI_ERR_ARG, "ctx is NULL");
  if (!xt || !xhat) return fail(DI_ERR_ARG, "xt and xhat must be non-NULL device pointers");
  if (batch < 1 || batch > c->max_batch) return fail(DI_ERR_ARG, "batch=%d outside [1, %d]", batch, c->max_batch);
  DevGuard dg_(c->device);
  if (!dg_.ok) return fail(DI_ERR_CUDA, "cudaSetDevice(%d) failed", c->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  void* x1 = const_cast<float*>(xt);
  if (c->prec == DI_PREC_BF16) {   // the bf16 path's x_tilde: the summed proxy rounded once (RNE)
    CUDA_TRY(di::launch_round_bf16(xt, c->xt, (size_t)batch * c->N, st));
    x1 = c->xt;
  }
  return run_stages(c, 1, 3, nullptr, 0, batch, x1, c->h1, c->h2, xhat, st);
}

di_status di_recover_host(di_ctx c, const void* y_host, long long ldy, int batch, float* xhat_host, void* stream) {
  if (!c) return fail(DI_ERR_ARG, "ctx is NULL");
  if (!y_host || !xhat_host) return fail(DI_ERR_ARG, "host buffers must be non-NULL");
  if (batch < 1 || batch > c->max_batch) return fail(DI_ERR_ARG, "batch=%d outside [1, %d]", batch, c->max_batch);
  if (ldy < c->m) return fail(DI_ERR_DIM, "ldy=%lld < m=%d", ldy, c->m);
  DevGuard dg_(c->device);
  if (!dg_.ok) return fail(DI_ERR_CUDA, "cudaSetDevice(%d) failed", c->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t ybytes = (size_t)batch * ldy * c->elt;
  if (ybytes > c->yhost_bytes) {
    if (c->yhost_dev) cudaFree(c->yhost_dev);
    c->yhost_dev = nullptr;
    c->yhost_bytes = 0;
    CUDA_TRY(cudaMalloc(&c->yhost_dev, ybytes));
    c->yhost_bytes = ybytes;
  }
  if (!c->xhost_dev) CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&c->xhost_dev), (size_t)c->max_batch * c->N * 4));
  if (!c->cstream) CUDA_TRY(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
  for (auto& e : c->cev)
    if (!e) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // Chunks shrinking geometrically by host_chunk_ratio r (4: 3B/4, 3B/16, ... while >= 128 images are left): the
  // device->host copy of x_hat for chunk k (copy stream) overlaps the kernels of chunk k+1 (caller's stream).  x_hat
  // leaves over PCIe ~4.7x faster than the path computes it (r02 e2e probe: 1.45 ms for 67 MB vs 6.9 ms), so a
  // chunk r = 4 times smaller still covers its predecessor's copy, and only the last, small chunk's copy is exposed.
  // Few chunks matter as much: every chunk pays the four kernels' ramp-up and drain (r = 2, the r01 plan, ran 6
  // chunks).  Chunks share the workspace: chunk k+1 only overwrites x_tilde/h1/h2, never the x_hat rows chunk k is
  // still copying out.
  int cuts[17] = {0};
  int nchunk = 0;
  if (batch >= 512) {
    const int r = c->host_chunk_ratio;
    // wave quantum (BF16 path): chunks of whole conv3 waves -- 2 images per item, one item per SM and 64-column
    // segment (k_conv3_r4) -- so the small chunks do not pay a partial last wave (lowrate: 2960 + 888 + 248 instead of
    // 3072 + 768 + 256, 14 instead of 16 conv3 waves per call)
    const int ncs = (c->n2 + 63) / 64;
    const int wq = (c->prec == DI_PREC_BF16 && c->host_waves) ? std::max(4, (2 * c->num_sms / ncs) & ~3) : 4;
    int left = batch;
    while (left > 0 && nchunk < 15) {
      int take = (left - left / r) & ~3;
      if (wq > 4) take = std::max(wq, (take + wq / 2) / wq * wq);
      if (left - take < 128 || nchunk == 14) take = left;
      cuts[nchunk + 1] = cuts[nchunk] + take;
      ++nchunk;
      left -= take;
    }
  } else {
    cuts[1] = batch, nchunk = 1;
  }
  // y: the first chunk's rows on the compute stream, the rest on the copy stream (overlapping chunk 0's kernels)
  const size_t y0bytes = (size_t)cuts[1] * ldy * c->elt;
  CUDA_TRY(cudaMemcpyAsync(c->yhost_dev, y_host, y0bytes, cudaMemcpyHostToDevice, st));
  if (nchunk > 1) {
    CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(c->yhost_dev) + y0bytes,
                             reinterpret_cast<const uint8_t*>(y_host) + y0bytes, ybytes - y0bytes, cudaMemcpyHostToDevice,
                             c->cstream));
    CUDA_TRY(cudaEventRecord(c->cev[16], c->cstream));
  }
  for (int k = 0; k < nchunk; ++k) {
    const int b0 = cuts[k], b1 = cuts[k + 1], nb = b1 - b0;
    if (k == 1) CUDA_TRY(cudaStreamWaitEvent(st, c->cev[16], 0));
    di_status s = run_stages(c, 0, 3, reinterpret_cast<const uint8_t*>(c->yhost_dev) + (size_t)b0 * ldy * c->elt, ldy,
                             nb, c->xt, c->h1, c->h2, c->xhost_dev + (size_t)b0 * c->N, st);
    if (s != DI_OK) return s;
    CUDA_TRY(cudaEventRecord(c->cev[k], st));
    CUDA_TRY(cudaStreamWaitEvent(c->cstream, c->cev[k], 0));
    CUDA_TRY(cudaMemcpyAsync(xhat_host + (size_t)b0 * c->N, c->xhost_dev + (size_t)b0 * c->N, (size_t)nb * c->N * 4,
                             cudaMemcpyDeviceToHost, c->cstream));
  }
  CUDA_TRY(cudaStreamSynchronize(c->cstream));
  CUDA_TRY(cudaStreamSynchronize(st));
  return DI_OK;
}

// stream key of synth/rng.py: stream_key(stream, sub = 0, seed)
static uint64_t sm64_mix_h(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}
static uint64_t stream_key(uint64_t stream, uint64_t seed) {
  uint64_t z = seed * 0x9E3779B97F4A7C15ull;
  z = sm64_mix_h(z + stream);
  return sm64_mix_h(z ^ (0ull * 0xBF58476D1CE4E5B9ull + 0x632BE59BD9B4E019ull));
}

di_status di_measure(di_ctx c, const float* x, int batch, void* y, long long ldy, void* stream) {
  if (!c) return fail(DI_ERR_ARG, "ctx is NULL");
  if (!x || !y) return fail(DI_ERR_ARG, "x and y must be non-NULL device pointers");
  if (batch < 1 || batch > c->max_batch) return fail(DI_ERR_ARG, "batch=%d outside [1, %d]", batch, c->max_batch);
  if (ldy < c->m) return fail(DI_ERR_DIM, "ldy=%lld < m=%d", ldy, c->m);
  DevGuard dg_(c->device);
  if (!dg_.ok) return fail(DI_ERR_CUDA, "cudaSetDevice(%d) failed", c->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (c->prec == DI_PREC_FP32) {
    CUDA_TRY(di::launch_measure_f32(x, c->phi_sense ? c->phi_sense : reinterpret_cast<const float*>(c->phi), c->m, c->N, batch,
                                    reinterpret_cast<float*>(y), ldy, st));
    return DI_OK;
  }
  const bool bf16 = c->prec == DI_PREC_BF16;
  const int kel = 128 / (int)c->elt;                // K elements per 128-B swizzle row
  if (!c->phi_rm) {                                 // Phi [m][npad] from the packed Phi^T, once
    c->npad = ((c->N + kel - 1) / kel) * kel;
    CUDA_TRY(cudaMalloc(&c->phi_rm, (size_t)c->m * c->npad * c->elt));
    CUDA_TRY(cudaMalloc(&c->xs, (size_t)c->max_batch * c->npad * c->elt));
    c->ws_bytes += (long long)((size_t)c->m * c->npad + (size_t)c->max_batch * c->npad) * c->elt;
    CUDA_TRY(di::launch_untranspose(c->phi, c->m, c->N, c->kpad, c->pxbn, c->npad, c->phi_rm, bf16, st));
  }
  CUDA_TRY(di::launch_stage_x(x, c->N, c->npad, batch, c->xs, bf16, st));
  // Y[B][m] = Xs[B][npad] . Phi_rm[m][npad]^T on the tcgen05 GEMM of the lifting layer (operand roles swapped)
  CUtensorMap tmA, tmB;
  di_status s = encode_2d(&tmA, c->xs, bf16, c->npad, batch, c->npad, kel, 128);
  if (s != DI_OK) return s;
  s = encode_2d(&tmB, c->phi_rm, bf16, c->npad, c->m, c->npad, kel, 256);
  if (s != DI_OK) return s;
  void* out = (ldy == c->m && (reinterpret_cast<uintptr_t>(y) & 15) == 0) ? y : c->ystage;
  CUDA_TRY(di::launch_proxy_tc(&tmA, &tmB, batch, c->m, c->npad / kel, out, !bf16, st));
  if (out != y)
    CUDA_TRY(cudaMemcpy2DAsync(y, (size_t)ldy * c->elt, out, (size_t)c->m * c->elt, (size_t)c->m * c->elt, batch,
                               cudaMemcpyDeviceToDevice, st));
  return DI_OK;
}

di_status di_add_noise(di_ctx c, void* y, long long ldy, int batch, double snr_db, unsigned long long seed,
                       void* stream) {
  if (!c) return fail(DI_ERR_ARG, "ctx is NULL");
  if (!y) return fail(DI_ERR_ARG, "y must be a non-NULL device pointer");
  if (batch < 1 || batch > c->max_batch) return fail(DI_ERR_ARG, "batch=%d outside [1, %d]", batch, c->max_batch);
  if (ldy < c->m) return fail(DI_ERR_DIM, "ldy=%lld < m=%d", ldy, c->m);
  if (std::isnan(snr_db)) return fail(DI_ERR_DOMAIN, "snr_db is NaN");
  if (std::isinf(snr_db) && snr_db > 0) return DI_OK;   // noiseless
  DevGuard dg_(c->device);
  if (!dg_.ok) return fail(DI_ERR_CUDA, "cudaSetDevice(%d) failed", c->device);
  CUDA_TRY(di::launch_add_noise(y, ldy, c->m, batch, snr_db, stream_key(5, seed), c->prec == DI_PREC_BF16,
                                reinterpret_cast<cudaStream_t>(stream)));
  return DI_OK;
}

di_status di_metrics(di_ctx c, const float* xhat, const float* x, int batch, double* out, void* stream) {
  if (!c) return fail(DI_ERR_ARG, "ctx is NULL");
  if (!xhat || !x || !out) return fail(DI_ERR_ARG, "NULL device pointer");
  if (batch < 1) return fail(DI_ERR_ARG, "batch=%d must be >= 1", batch);
  DevGuard dg_(c->device);
  if (!dg_.ok) return fail(DI_ERR_CUDA, "cudaSetDevice(%d) failed", c->device);
  CUDA_TRY(di::launch_metrics(xhat, x, c->N, batch, out, reinterpret_cast<cudaStream_t>(stream)));
  return DI_OK;
}

// ---------------------------------------------------------------------------------------------- training
// the tensor-core weight images from the parameters: the forward's (TF32 fp32 images or BF16 bf16 images) and the
// backward's (layer-3 dgrad bank, bf16 layer-2 dgrad blocks)
static cudaError_t repack_tc(di_ctx c, cudaStream_t st) {
  const int flip = !(c->flags & DI_FLAG_XCORR);
  if (c->prec == DI_PREC_BF16) {
    cudaError_t e = di::launch_repack_tf32(c->params, flip, nullptr, nullptr, nullptr, c->wpd3, c->wp2db, st);
    if (e != cudaSuccess) return e;
    return di::launch_repack_bf16(c->params, flip, c->wp1, c->wp2, c->wp3, st);
  }
  return di::launch_repack_tf32(c->params, flip, reinterpret_cast<float*>(c->wp1), reinterpret_cast<float*>(c->wp2t),
                                reinterpret_cast<float*>(c->wp3), c->wpd3, c->wp2db, st);
}

static di_status train_alloc(di_ctx c) {
  if (c->dxh) return DI_OK;
  const size_t B = (size_t)c->max_batch, N = (size_t)c->N;
  auto al = [&](auto** p, size_t bytes) -> di_status {
    CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(p), bytes));
    c->ws_bytes += (long long)bytes;
    return DI_OK;
  };
  di_status s;
  if ((s = al(&c->wt2, (size_t)C2 * K * K * C1 * 4)) != DI_OK) return s;
  if ((s = al(&c->wt3, (size_t)K * K * C2 * 4)) != DI_OK) return s;
  if ((s = al(&c->xh_ws, B * N * 4)) != DI_OK) return s;
  if ((s = al(&c->dxh, B * N * 4)) != DI_OK) return s;
  if ((s = al(&c->dh2, B * N * C2 * 4)) != DI_OK) return s;
  if ((s = al(&c->dh1, B * N * C1 * 4)) != DI_OK) return s;
  const size_t pw = std::max({(size_t)(di::WGRAD_CHUNKS / 4) * C2 * K * K, (size_t)(di::WGRAD_CHUNKS / 32) * C2 * C1 * K * K,
                              (size_t)(di::WGRAD_CHUNKS / 4) * C1 * K * K});
  if ((s = al(&c->part_w, pw * 4)) != DI_OK) return s;
  if ((s = al(&c->part_b, (size_t)di::WGRAD_CHUNKS * C1 * 4)) != DI_OK) return s;
  if ((s = al(&c->loss_img, B * 8)) != DI_OK) return s;
  // backward layouts (and the forward ones, identical to di_create's) from the parameters
  CUDA_TRY(di::launch_sgd_repack(c->params, nullptr, c->vel, di::N_PARAMS, 0.f, 0.f, !(c->flags & DI_FLAG_XCORR),
                                 c->wx1, c->wx2, c->wx3, c->wt2, c->wt3, c->b1, c->b2, c->b3, 0));
  if (c->prec != DI_PREC_FP32) {
    const bool bf = c->prec == DI_PREC_BF16;
    CUDA_TRY(di::setup_conv2_tc(c->n2));   // the bf16 layer-2 kernel also runs the layer-2 data gradient
    if (!bf && (s = al(&c->h1b, B * N * C1 * 2)) != DI_OK) return s;   // (BF16: h1 itself is bf16)
    if ((s = al(&c->dg2b, B * N * C2 * 2)) != DI_OK) return s;
    if ((s = al(&c->dh1b, B * N * C1 * 2)) != DI_OK) return s;
    if ((s = al(&c->part_w2, std::max(di::wgrad2_tc_part_floats(c->num_sms), di::wgrad13_tc_part_floats(c->num_sms)) * 4)) != DI_OK)
      return s;
    if ((s = encode_wg2(&c->tmH1b, bf ? c->h1 : c->h1b, c->max_batch, c->n1, c->n2, 64, di::wgrad2_tc_h_box_rows())) !=
        DI_OK)
      return s;
    if ((s = encode_wg2(&c->tmDG2b, c->dg2b, c->max_batch, c->n1, c->n2, 32, di::wgrad2_tc_g_box_rows())) != DI_OK)
      return s;
    CUDA_TRY(di::setup_wgrad2_tc(c->n2));
    CUDA_TRY(di::setup_wgrad13_tc(c->n2));
    // the layer-3 wgrad's bf16 h2 strip: BF16 reads h2 itself, TF32 a bf16 copy of h2 made in the (then idle) h1b
    if ((s = encode_wg2(&c->tmH2w, bf ? c->h2 : c->h1b, c->max_batch, c->n1, c->n2, 32, di::wgrad3_tc_h_box_rows())) !=
        DI_OK)
      return s;
    if ((s = encode_wg2(&c->tmD1w, c->dh1b, c->max_batch, c->n1, c->n2, 64, di::wgrad1_tc_d_box_rows())) != DI_OK)
      return s;
    if ((s = al(reinterpret_cast<uint8_t**>(&c->wp2db), (size_t)di::DG2_KBLOCKS * 8192)) != DI_OK) return s;
    if ((s = encode_dg2b_strip(&c->tmDG2s, c->dg2b, c->max_batch, c->n1, c->n2)) != DI_OK) return s;
    if (c->n2 % 4 == 0) {   // the conv1 TF32 strip map over dG3 (16-B row stride)
      if ((s = al(&c->wpd3, (size_t)11 * 4096)) != DI_OK) return s;
      if ((s = encode_xt(&c->tmDX, c->dxh, c->max_batch, c->n1, c->n2, true)) != DI_OK) return s;
      c->has_tmDX = true;
    }
    CUDA_TRY(repack_tc(c, 0));
  }
  CUDA_TRY(cudaDeviceSynchronize());
  return DI_OK;
}

// custom stacks (NEXT-3): the forward keeps every hidden layer's output (fp32), the backward runs the generic SIMT
// weight / data gradient kernels per layer
static di_status train_alloc_stack(di_ctx c) {
  if (c->dxh) return DI_OK;
  const size_t B = (size_t)c->max_batch, N = (size_t)c->N;
  auto al = [&](auto** p, size_t bytes) -> di_status {
    CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(p), bytes));
    c->ws_bytes += (long long)bytes;
    return DI_OK;
  };
  di_status s;
  const int L = (int)c->stack.size();
  int cmax = 1;
  size_t pw = 0, pb = 0;
  for (int i = 0; i < L; ++i) {
    di_ctx_s::Layer& l = c->stack[i];
    if (i < L - 1 && (s = al(&l.keep, B * N * l.cout * 4)) != DI_OK) return s;
    if (i > 0) {
      if ((s = al(&l.wt, (size_t)l.cout * l.cin * K * K * 4)) != DI_OK) return s;
      cmax = std::max(cmax, l.cin);
    }
    if (!l.b) {   // trainable biases need storage even when created zero (k_conv1_tc reads 64)
      const size_t nbias = (c->prec == DI_PREC_BF16 && i == 0) ? 64 : (size_t)l.cout;
      if ((s = al(&l.b, nbias * 4)) != DI_OK) return s;
      CUDA_TRY(cudaMemset(l.b, 0, nbias * 4));
    }
    pw = std::max(pw, di::wgrad_layer_part_floats(l.cin, l.cout));
    pb = std::max(pb, di::wgrad_layer_partb_floats(l.cin, l.cout));
  }
  if (c->prec == DI_PREC_BF16 && (s = al(&c->keep_x, B * N * 4)) != DI_OK) return s;
  if ((s = al(&c->xh_ws, B * N * 4)) != DI_OK) return s;
  if ((s = al(&c->dxh, B * N * 4)) != DI_OK) return s;
  if ((s = al(&c->dA, B * N * cmax * 4)) != DI_OK) return s;
  if ((s = al(&c->dB, B * N * cmax * 4)) != DI_OK) return s;
  if ((s = al(&c->part_w, pw * 4)) != DI_OK) return s;
  if ((s = al(&c->part_b, pb * 4)) != DI_OK) return s;
  if ((s = al(&c->loss_img, B * 8)) != DI_OK) return s;
  return DI_OK;
}

static di_status train_check(di_ctx c) {
  if (!c) return fail(DI_ERR_ARG, "ctx is NULL");
  if (!c->params) return fail(DI_ERR_ARG, "training needs a context with per-channel (or zero) biases");
  if (!c->stack.empty()) return train_alloc_stack(c);
  if (c->prec == DI_PREC_BF16 && c->n2 % 4 != 0)
    return fail(DI_ERR_ARG, "BF16 training needs n2 %% 4 == 0 (the layer-3 data gradient's strip map)");
  if (!c->b1 || !c->b2 || !c->b3) {   // trainable biases need storage even when created zero
    if (!c->b1) CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&c->b1), C1 * 4));
    if (!c->b2) CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&c->b2), C2 * 4));
    if (!c->b3) CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&c->b3), 4));
  }
  return train_alloc(c);
}

static di_status train_grad_stack(di_ctx c, const void* y, long long ldy, const float* x_true, int batch, double scale,
                                  float* grads, double* loss, cudaStream_t st) {
  const int L = (int)c->stack.size();
  const int flip = !(c->flags & DI_FLAG_XCORR);
  const size_t npix = (size_t)batch * c->N;
  // backward banks from the current parameters (cheap; always consistent with params)
  for (int i = 1; i < L; ++i) {
    const di_ctx_s::Layer& l = c->stack[i];
    CUDA_TRY(di::launch_repack_layer(c->params + l.woff, nullptr, l.cin, l.cout, flip, nullptr, l.wt, nullptr, st));
  }
  // forward through the context's own kernels, keeping x_tilde and every hidden output as fp32
  int launches = 0;
  di_status s = run_proxy(c, y, ldy, batch, c->xt, false, st, launches);
  if (s != DI_OK) return s;
  s = run_stack(c, batch, c->xt, c->xh_ws, st, launches, true);
  if (s != DI_OK) return s;
  const float* xt32 = reinterpret_cast<const float*>(c->xt);
  if (c->prec == DI_PREC_BF16) {
    CUDA_TRY(di::launch_bf16_to_f32(c->xt, 1, 1, npix, c->keep_x, st));
    xt32 = c->keep_x;
  }
  // loss and dL/dx_hat, the last layer's ReLU' under DI_FLAG_FINAL_RELU
  CUDA_TRY(di::launch_loss_grad(c->xh_ws, x_true, c->N, batch, scale, c->dxh, c->loss_img, loss, st));
  if (c->flags & DI_FLAG_FINAL_RELU) CUDA_TRY(di::launch_dgrad_mask(c->dxh, c->xh_ws, npix, st));
  const size_t nw = (size_t)c->nparams - (c->stack.back().boff + c->stack.back().cout);
  float* g = c->dxh;
  for (int i = L - 1; i >= 0; --i) {
    const di_ctx_s::Layer& l = c->stack[i];
    const float* X = i == 0 ? xt32 : c->stack[i - 1].keep;
    CUDA_TRY(di::launch_wgrad_layer(l.cin, l.cout, X, g, batch, c->n1, c->n2, c->part_w, c->part_b, flip,
                                    grads + l.woff, grads + nw + l.boff, st));
    if (i > 0) {   // dX = [X > 0] * (dG correlated with the rotated, transposed bank)
      float* dX = g == c->dA ? c->dB : c->dA;
      CUDA_TRY(di::launch_dgrad_simt(l.cin, l.cout, g, l.wt, X, dX, batch, c->n1, c->n2, st));
      g = dX;
    }
  }
  return DI_OK;
}

di_status di_train_grad(di_ctx c, const void* y, long long ldy, const float* x_true, int batch, double scale,
                        float* grads, double* loss, void* stream) {
  if (!c) return fail(DI_ERR_ARG, "ctx is NULL");
  DevGuard dg_(c->device);   // train_check allocates on the context's device
  if (!dg_.ok) return fail(DI_ERR_CUDA, "cudaSetDevice(%d) failed", c->device);
  di_status s = train_check(c);
  if (s != DI_OK) return s;
  if (!y || !x_true || !grads || !loss) return fail(DI_ERR_ARG, "NULL device pointer");
  if (batch < 1 || batch > c->max_batch) return fail(DI_ERR_ARG, "batch=%d outside [1, %d]", batch, c->max_batch);
  if (ldy < c->m) return fail(DI_ERR_DIM, "ldy=%lld < m=%d", ldy, c->m);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!c->stack.empty()) return train_grad_stack(c, y, ldy, x_true, batch, scale, grads, loss, st);
  const int flip = !(c->flags & DI_FLAG_XCORR);
  const int relu3 = (c->flags & DI_FLAG_FINAL_RELU) ? 1 : 0;
  // forward, keeping x_tilde, h1, h2 (post-ReLU) in the workspace
  s = run_stages(c, 0, 3, y, ldy, batch, c->xt, c->h1, c->h2, c->xh_ws, st);
  if (s != DI_OK) return s;
  const size_t n1w = (size_t)C1 * K * K, n2w = (size_t)C2 * C1 * K * K, n3w = (size_t)C2 * K * K;
  float* gb = grads + n1w + n2w + n3w;
  CUDA_TRY(di::launch_loss_grad(c->xh_ws, x_true, c->N, batch, scale, c->dxh, c->loss_img, loss, st));
  if (relu3)   // dG3 = dx_hat * ReLU'(x_hat): the mask is applied by the layer-3 dgrad input convention below
    CUDA_TRY(di::launch_dgrad_mask(c->dxh, c->xh_ws, (size_t)batch * c->N, st));
  const float* xt = reinterpret_cast<const float*>(c->xt);
  const float* h1 = reinterpret_cast<const float*>(c->h1);
  const float* h2 = reinterpret_cast<const float*>(c->h2);
  const bool tc = c->prec != DI_PREC_FP32;   // tensor-core backward (k_conv2_tc<32, 64>, k_wgrad*_tc, dgrad3)
  const bool bf = c->prec == DI_PREC_BF16;   // BF16 contexts: x_tilde, h1, h2 are bf16
  if (tc) {   // bf16 h2 operand by TMA (TF32: rounded into h1b first -- the kernel rounds to bf16 either way)
    if (!bf) CUDA_TRY(di::launch_to_bf16(h2, c->h1b, (size_t)batch * c->N * C2, st));
    CUDA_TRY(di::launch_wgrad3_tc(bf ? c->h2 : c->h1b, c->dxh, batch, c->n1, c->n2, c->part_w2, c->part_b, flip,
                                  grads + n1w + n2w, gb + C1 + C2, c->num_sms, st, true, &c->tmH2w));
  } else
    CUDA_TRY(di::launch_wgrad(3, h2, c->dxh, batch, c->n1, c->n2, c->part_w, c->part_b, flip, grads + n1w + n2w,
                              gb + C1 + C2, st));
  const bool dg3tc = tc && c->has_tmDX;   // tensor-core dgrad3 writes bf16 dG2 and the layer-2 bias gradient itself
  if (dg3tc)
    CUDA_TRY(di::launch_dgrad3_tf32(&c->tmDX, c->wpd3, c->h2, c->dg2b, c->part_b, gb + C1, batch, c->n1, c->n2,
                                    c->num_sms, st, bf));
  else
    CUDA_TRY(di::launch_dgrad3_f32(c->dxh, c->wt3, h2, c->dh2, batch, c->n1, c->n2, st));
  if (tc) {   // bf16 operands, tcgen05 MN-major contraction over pixels (k_wgrad2_tc.cu)
    const size_t npix = (size_t)batch * c->N;
    if (!dg3tc) {
      CUDA_TRY(di::launch_dg2_bf16(c->dh2, npix, c->dg2b, c->part_b, st));
      CUDA_TRY(di::launch_bias_reduce(c->part_b, di::WGRAD_CHUNKS, C2, gb + C1, st));
    }
    if (!bf) CUDA_TRY(di::launch_to_bf16(h1, c->h1b, npix * C1, st));   // (BF16: h1 is the bf16 operand)
    CUDA_TRY(di::launch_wgrad2_tc(&c->tmH1b, &c->tmDG2b, batch, c->n1, c->n2, c->part_w2, flip, grads + n1w,
                                  c->num_sms, st));
  } else {
    CUDA_TRY(di::launch_wgrad(2, h1, c->dh2, batch, c->n1, c->n2, c->part_w, c->part_b, flip, grads + n1w, gb + C1,
                              st));
  }
  if (tc)   // bf16 operands from the dG2 copy made for wgrad2: twice the TF32 MMA rate
    CUDA_TRY(di::launch_dgrad2_bf16(&c->tmDG2s, c->wp2db, bf ? c->h1 : c->h1b, batch, c->n1, c->n2, c->dh1b,
                                    c->num_sms, st));
  else
    CUDA_TRY(di::launch_dgrad2_f32(c->dh2, c->wt2, h1, c->dh1, batch, c->n1, c->n2, st));
  if (tc)
    CUDA_TRY(di::launch_wgrad1_tc(c->xt, c->dh1b, batch, c->n1, c->n2, c->part_w2, c->part_b, flip, grads, gb,
                                  c->num_sms, st, bf, &c->tmD1w));
  else
    CUDA_TRY(di::launch_wgrad(1, xt, c->dh1, batch, c->n1, c->n2, c->part_w, c->part_b, flip, grads, gb, st));
  return DI_OK;
}

// custom stacks: the SGD step on the device; the forward images re-derived from the parameters -- on the device for
// FP32 contexts (SIMT layout), on the host with di_create's packers for TF32 / BF16 (the tensor-core images of every
// layer type; one synchronisation of `st` per step)
static di_status sgd_stack(di_ctx c, const float* grads, double lr, double momentum, cudaStream_t st) {
  CUDA_TRY(di::launch_sgd(c->params, grads, c->vel, (int)c->nparams, (float)lr, (float)momentum, st));
  const int L = (int)c->stack.size();
  const bool xc = (c->flags & DI_FLAG_XCORR) != 0;
  const size_t nw = (size_t)c->nparams - (c->stack.back().boff + c->stack.back().cout);
  if (c->prec == DI_PREC_FP32) {
    for (auto& l : c->stack)
      CUDA_TRY(di::launch_repack_layer(c->params + l.woff, c->params + nw + l.boff, l.cin, l.cout, !xc, l.wx, nullptr,
                                       l.b, st));
    return DI_OK;
  }
  std::vector<float> prm((size_t)c->nparams);
  CUDA_TRY(cudaMemcpyAsync(prm.data(), c->params, prm.size() * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  for (int i = 0; i < L; ++i) {
    di_ctx_s::Layer& l = c->stack[i];
    const auto img = pack_stack_layer(c->prec, i, L, xcorr_taps(prm.data() + l.woff, l.cout, l.cin, xc, false), l.cin,
                                      l.cout);
    CUDA_TRY(cudaMemcpyAsync(l.wp, img.data(), img.size(), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(l.b, prm.data() + nw + l.boff, (size_t)l.cout * 4, cudaMemcpyHostToDevice, st));
  }
  CUDA_TRY(cudaStreamSynchronize(st));   // the host images are released on return
  return DI_OK;
}

di_status di_sgd_step(di_ctx c, const float* grads, double lr, double momentum, void* stream) {
  if (!c) return fail(DI_ERR_ARG, "ctx is NULL");
  DevGuard dg_(c->device);   // train_check allocates on the context's device
  if (!dg_.ok) return fail(DI_ERR_CUDA, "cudaSetDevice(%d) failed", c->device);
  di_status s = train_check(c);
  if (s != DI_OK) return s;
  if (!grads) return fail(DI_ERR_ARG, "grads is NULL");
  if (!(lr >= 0.0) || !(momentum >= 0.0 && momentum < 1.0)) return fail(DI_ERR_DOMAIN, "lr >= 0, 0 <= momentum < 1");
  if (!c->stack.empty()) return sgd_stack(c, grads, lr, momentum, reinterpret_cast<cudaStream_t>(stream));
  CUDA_TRY(di::launch_sgd_repack(c->params, grads, c->vel, di::N_PARAMS, (float)lr, (float)momentum,
                                 !(c->flags & DI_FLAG_XCORR), c->wx1, c->wx2, c->wx3, c->wt2, c->wt3, c->b1, c->b2,
                                 c->b3, reinterpret_cast<cudaStream_t>(stream)));
  if (c->prec != DI_PREC_FP32) CUDA_TRY(repack_tc(c, reinterpret_cast<cudaStream_t>(stream)));
  return DI_OK;
}

di_status di_get_params(di_ctx c, float* params, void* stream) {
  if (!c || !params) return fail(DI_ERR_ARG, "NULL argument");
  if (!c->params) return fail(DI_ERR_ARG, "not a trainable (FP32, per-channel bias) context");
  DevGuard dg_(c->device);
  CUDA_TRY(cudaMemcpyAsync(params, c->params, (size_t)c->nparams * 4, cudaMemcpyDeviceToDevice,
                           reinterpret_cast<cudaStream_t>(stream)));
  return DI_OK;
}

long long di_num_params(void) { return di::N_PARAMS; }

long long di_ctx_num_params(di_ctx c) { return c ? c->nparams : 0; }

di_status di_destroy(di_ctx c) {
  if (!c) return DI_OK;
  DevGuard dg_(c->device);
  cudaDeviceSynchronize();
  free_ctx(c);
  return DI_OK;
}

di_status di_get_info(di_ctx c, di_info* info) {
  if (!c || !info) return fail(DI_ERR_ARG, "NULL argument");
  info->m = c->m, info->n1 = c->n1, info->n2 = c->n2, info->max_batch = c->max_batch;
  info->precision = c->prec, info->flags = c->flags;
  info->launches_per_recover = c->last_launches ? c->last_launches : 4;
  info->workspace_bytes = c->ws_bytes;
  const bool bf16 = c->prec == DI_PREC_BF16;
  info->stage_kernels[0] = c->prec == DI_PREC_FP32 ? "k_proxy_f32" : (bf16 ? "k_proxy_tc<bf16>" : "k_proxy_tc<tf32>");
  info->stage_kernels[1] = bf16 ? "k_conv1_tc" : (c->prec == DI_PREC_TF32 && c->has_tmX ? "k_conv1_tf32" : "k_conv_wide<conv1>");
  info->stage_kernels[2] = bf16 ? "k_conv2_tc" : (c->prec == DI_PREC_TF32 ? "k_conv2_tf32" : "k_conv_wide<conv2,f32>");
  info->stage_kernels[3] = c->prec != DI_PREC_FP32 ? "k_conv3_tc" : "k_conv3";
  return DI_OK;
}

di_status di_set_profiling(di_ctx c, int enable) {
  if (!c) return fail(DI_ERR_ARG, "ctx is NULL");
  c->profiling = enable != 0;
  return DI_OK;
}

di_status di_stage_times(di_ctx c, float ms[4], int* calls, int reset) {
  if (!c || !ms) return fail(DI_ERR_ARG, "NULL argument");
  if (c->ev_used > 0) {
    CUDA_TRY(cudaEventSynchronize(c->evpool[c->ev_used - 1][4]));
    for (int k = 0; k < c->ev_used; ++k) {
      for (int i = 0; i < 4; ++i) {
        float t = 0.f;
        if (cudaEventElapsedTime(&t, c->evpool[k][i], c->evpool[k][i + 1]) == cudaSuccess) c->stage_ms[i] += t;
      }
      c->prof_calls++;
    }
    c->ev_used = 0;
  }
  for (int i = 0; i < 4; ++i) ms[i] = c->stage_ms[i];
  if (calls) *calls = c->prof_calls;
  if (reset) {
    for (int i = 0; i < 4; ++i) c->stage_ms[i] = 0.f;
    c->prof_calls = 0;
  }
  return DI_OK;
}

di_status di_debug_stage(di_ctx c, int stage, const void* in, void* out, int batch, void* stream) {
  if (!c) return fail(DI_ERR_ARG, "ctx is NULL");
  if (stage < 0 || stage > 3) return fail(DI_ERR_ARG, "stage=%d outside [0,3]", stage);
  if (!in || !out) return fail(DI_ERR_ARG, "NULL buffer");
  if (batch < 1 || batch > c->max_batch) return fail(DI_ERR_ARG, "batch=%d outside [1, %d]", batch, c->max_batch);
  if (stage > 0 && !c->stack.empty()) return fail(DI_ERR_ARG, "per-stage hooks are for the paper's stack");
  DevGuard dg_(c->device);
  if (!dg_.ok) return fail(DI_ERR_CUDA, "cudaSetDevice(%d) failed", c->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (stage) {
    case 0: return run_stages(c, 0, 0, in, c->m, batch, out, nullptr, nullptr, nullptr, st);
    case 1: return run_stages(c, 1, 1, nullptr, 0, batch, const_cast<void*>(in), out, nullptr, nullptr, st);
    case 2: return run_stages(c, 2, 2, nullptr, 0, batch, nullptr, const_cast<void*>(in), out, nullptr, st);
    default:
      return run_stages(c, 3, 3, nullptr, 0, batch, nullptr, nullptr, const_cast<void*>(in),
                        reinterpret_cast<float*>(out), st);
  }
}

di_status di_debug_get_phi(di_ctx c, void* host_out, long long bytes) {
  if (!c || !host_out) return fail(DI_ERR_ARG, "NULL argument");
  const size_t need = (size_t)c->m * c->N * c->elt;
  if ((size_t)bytes < need) return fail(DI_ERR_DIM, "need %zu bytes", need);
  DevGuard dg_(c->device);
  if (c->prec == DI_PREC_FP32) {
    CUDA_TRY(cudaMemcpy(host_out, c->phi, need, cudaMemcpyDeviceToHost));
    return DI_OK;
  }
  // tile-blocked Phi^T -> Phi [m][N]
  std::vector<uint8_t> t(di::phiT_blk_elems(c->N, c->kpad, c->pxbn) * c->elt);
  CUDA_TRY(cudaMemcpy(t.data(), c->phi, t.size(), cudaMemcpyDeviceToHost));
  uint8_t* o = reinterpret_cast<uint8_t*>(host_out);
  const int kel = 128 / (int)c->elt;
  for (int i = 0; i < c->m; ++i)
    for (int j = 0; j < c->N; ++j)
      std::memcpy(o + ((size_t)i * c->N + j) * c->elt, t.data() + di::phiT_blk_index(j, i, c->kpad, kel, c->pxbn) * c->elt,
                  c->elt);
  return DI_OK;
}

}  // extern "C"
