// kernels.cuh -- launch entry points of the DeepInverse kernels (internal; the public ABI is
// include/deepinverse.h).  All launches are asynchronous on the given stream.
#pragma once
// Instrumentation and geometry overrides exist only in the experiment library (build.py: DI_NVCC_EXTRA builds
// libdeepinverse_exp.so with -DDI_EXPERIMENT_BUILD); the product library cannot be compiled with them.
#if !defined(DI_EXPERIMENT_BUILD) && (defined(DI_PROF_CONV1) || defined(DI_PROF_CONV2) || defined(DI_PROF_CONV3) || \
                                      defined(DI_C2_ROWS) || defined(DI_C2_WSTAGES) || defined(DI_C3R_PF) || \
                                      defined(DI_C3R_NSL) || defined(DI_EXP_GENERIC_SMEM))
#error "experiment macros need DI_EXPERIMENT_BUILD (build.py routes them to libdeepinverse_exp.so)"
#endif
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace di {

// conv2 tensor-core geometry (k_conv2_tc.cu)
#ifndef DI_C2_ROWS
#define DI_C2_ROWS 6
#endif
constexpr int C2_ROWS = DI_C2_ROWS;         // output rows per work unit
constexpr int C2_KBLOCKS = 33;              // 11 tap rows x 3 column-tap groups of 4
constexpr int C2_KBLOCK_BYTES = 128 * 128;  // 128 rows (4 taps x 32 filters) x 64 ch x bf16

// conv1 / conv3 tensor-core geometry (k_conv13_tc.cu)
constexpr int C1TC_ROWS = 16;               // conv1 output rows per work unit
constexpr int C3TC_ROWS = 6;                // conv3 output rows per work unit

// stage 0: lifting layer x_tilde = Phi^T y
// Row-sharded Phi (NEXT-4): the fp32 partial of image b goes straight to the staging buffer of the rank that owns
// b's batch block: slots[b / nb] + (rank * nb + b % nb) * N (slots[r] may be a peer-mapped pointer into rank r's
// memory); world = 0 disables the scatter
struct ProxyScatter {
  float* slots[8];
  int world, rank, nb;
};
cudaError_t setup_proxy_tc();
size_t proxy_tc_smem_bytes();
// tmPt: a 2-D map over a row-major [N][K] operand (box 128 B x 256 rows), or with b_blocked a 3-D map over the
// tile-blocked Phi^T of the lifting layer (phiT_blk_index: box = one contiguous 32-KB (N-tile, K-block) block)
cudaError_t launch_proxy_tc(const CUtensorMap* tmY, const CUtensorMap* tmPt, int batch, int N, int kblocks,
                            void* xt, bool tf32, cudaStream_t st, bool out_f32 = false,
                            const ProxyScatter* sc = nullptr, bool b_blocked = false, int bn = 256);
// pixel-tile width of the lifting GEMM (256, or 224 when that fills the SM waves better for max_batch)
int proxy_tile_width(long long N, int max_batch, bool bf16, int num_sms);
// the lifting GEMM on CTA pairs (cta_group::2, M = 256 images): bf16 x_tilde; tmPh = half-block Phi^T boxes
cudaError_t setup_proxy_pair();
cudaError_t launch_proxy_pair(const CUtensorMap* tmY, const CUtensorMap* tmPh, int batch, int N, int kblocks, void* xt,
                              int bn, cudaStream_t st);
// Tile-blocked Phi^T (BF16 / TF32 contexts): element (pixel j, measurement i) of [N-tile j / tr][K-block i / kel]
// [j % tr][i % kel], kel = 128 B / element size, tr = the GEMM's pixel-tile width; one (N-tile, K-block) block is
// the tr x 128 B the proxy GEMM stages per K-block, contiguous in HBM (full DRAM pages instead of tr strided 128-B
// rows).  Size: ceil(N / tr) * tr * kpad.
__host__ __device__ inline size_t phiT_blk_index(long long j, int i, int kpad, int kel, int tr) {
  return (((size_t)(j / tr) * (size_t)(kpad / kel) + (size_t)(i / kel)) * tr + (size_t)(j % tr)) * kel + i % kel;
}
__host__ __device__ inline size_t phiT_blk_elems(long long N, int kpad, int tr) {
  return (size_t)((N + tr - 1) / tr) * tr * kpad;
}
// rows of a local fp32 partial [batch][N] to the owners' slots (FP32 contexts); the owner's fixed-order slot sum
// staging [world][nb][N] -> x_tilde [nb][N] (fp32, or RNE bf16 when bf16)
cudaError_t launch_scatter_rows(const float* src, int batch, int N, const ProxyScatter* sc, cudaStream_t st);
cudaError_t launch_reduce_slots(const float* staging, int world, int nb, int N, void* out, bool bf16, cudaStream_t st);
cudaError_t launch_round_bf16(const float* src, void* dst, size_t n, cudaStream_t st);
cudaError_t launch_proxy_f32(const float* y, long long ldy, const float* phi, int m, int N, int batch, float* xt,
                             cudaStream_t st);
cudaError_t launch_pack_phiT(const float* phi, int m, int N, int kpad, int tr, void* out, bool bf16, cudaStream_t st);
cudaError_t launch_stage_y(const void* y, long long ldy, int m, int kpad, int batch, void* out, bool bf16,
                           cudaStream_t st);

// stage 1: conv layer 1 (1 -> 64, ReLU)
cudaError_t launch_conv1_simt(const void* xt, bool bf16, const float* wx, const float* bias, int fullmap, void* h1,
                              int batch, int n1, int n2, cudaStream_t st);

cudaError_t setup_conv13_tc(int n2);
int conv1_tc_box_rows();
int conv1_tc_box_cols(int n2);
// tmX: 3-D tensor map of x_tilde (n2 % 8 == 0) for the TMA strip path, or nullptr for the gather path
cudaError_t launch_conv1_tc(const CUtensorMap* tmX, const CUtensorMap* tmS, const void* xt, const void* w1pack,
                            const float* bias, int fullmap, void* h1, int batch, int n1, int n2, int num_sms,
                            cudaStream_t st);

int conv1_tf32_box_rows();
// TF32 mode: tmX = 3-D map of the fp32 x_tilde (n2 % 4 == 0), box (P + 8) x (8 + 10) x 1
cudaError_t launch_conv1_tf32(const CUtensorMap* tmX, const void* w1pack, const float* bias, int fullmap, float* h1,
                              int batch, int n1, int n2, int num_sms, cudaStream_t st);

// stage 2: conv layer 2 (64 -> 32, ReLU)
cudaError_t setup_conv2_tc(int n2);
size_t conv2_tc_smem_bytes(int n2);
// mixed row-block heights (n1 = ntall 7-row + 6-row blocks) when they cut the MMA tiles per image; 0: uniform
int conv2_tc_tall_blocks(int n1, int n2);
int conv2_tc_box_rows(int n1, int n2, int mixed);
int conv2_tc_box_cols(int n2);
int dgrad2_bf16_box_rows();
// custom stacks, BF16: interior C_in -> C_out layers on k_conv2_tc (bias + ReLU), strip box rows per C_in
int convg_tc_box_rows(int cin);
cudaError_t setup_convg_tc(int n2);
cudaError_t launch_convg_tc(int cin, int cout, const CUtensorMap* tm, const void* wpack, const float* bias, int batch,
                            int n1, int n2, void* out, int num_sms, cudaStream_t st);
cudaError_t launch_conv2_tc(const CUtensorMap* tmH1, const void* wpack, const float* bias, int fullmap, int batch,
                            int n1, int n2, void* h2, int num_sms, cudaStream_t st, int cluster,
                            int balanced = 1, int mixed = 1);
size_t conv2_tf32_smem_bytes(int n2);
int conv2_tf32_box_rows();
int conv_tf32_box_cols(int n2);   // strip pitch of k_conv_tf32 (n2 + 5, or 74 with several column segments)
int wgrad_box_cols(int n2);       // strip pitch W + 10 of the layer-2 wgrad / wgrad1 / wgrad3 operands
cudaError_t setup_conv2_tf32(int n2);
// generic TF32 layer C_in -> C_out, (C_in, C_out) in {32, 64}^2, bias + ReLU (deeper / wider stacks, NEXT-3);
// wpack: convg_tf32_kblocks(cin, cout) blocks of 16 KB (api.cu conv_tf32_pack)
int convg_tf32_kblocks(int cin, int cout);
cudaError_t launch_convg_tf32(int cin, int cout, const CUtensorMap* tmIn, const void* wpack, const float* bias,
                              int batch, int n1, int n2, float* out, int num_sms, cudaStream_t st);
cudaError_t launch_conv2_tf32(const CUtensorMap* tmH1, const void* wpack, const float* bias, int fullmap, int batch,
                              int n1, int n2, float* h2, int num_sms, cudaStream_t st);
cudaError_t launch_conv2_simt_f32(const float* h1, const float* wx, const float* bias, int fullmap, float* h2,
                                  int batch, int n1, int n2, cudaStream_t st);

// stage 3: conv layer 3 (32 -> 1, optional ReLU)
cudaError_t launch_conv3_simt(const void* h2, bool bf16, const float* wx, const float* bias, int fullmap, int relu,
                              float* xhat, int batch, int n1, int n2, cudaStream_t st);

int conv3_tc_box_rows();
// bf16 conv layer 3 with C3R_RP output rows stacked in M (k_conv3_r4.cu); tpack: the tap-row stack T (api.cu
// conv3_r4_pack): C3R_NENT entries T[C3R_IMIN + e] of C3R_ES rows (column taps, 11 valid) x 32 channels bf16
constexpr int C3R_RP = 11;                      // output rows per pass (= per unit)
constexpr int C3R_ES = 11;                      // M rows per output row: the 11 column taps (121 of 128 rows used)
constexpr int C3R_NWIN = C3R_RP + 10;           // windows (strip rows) per pass
constexpr int C3R_IMIN = 11 - C3R_NWIN;
constexpr int C3R_NENT = C3R_NWIN + C3R_RP - 1;
int conv3_r4_box_rows();
int conv3_r4_box_cols(int n2);   // positions per image of a strip row (W + 10 rounded up to 16)
int conv3_r4_tpack_bytes();
cudaError_t setup_conv3_r4(int n2);
// xtrue (optional, DEVICE [batch][n1][n2] fp32): metrics fused into the epilogue -> metrics [3][batch] (PSNR, NMSE,
// success as di_metrics) through the per-item partial buffer mpart (conv3_r4_metrics_part_bytes)
cudaError_t launch_conv3_r4(const CUtensorMap* tmH2, const void* tpack, const float* bias, int fullmap, int relu,
                            float* xhat, int batch, int n1, int n2, int num_sms, cudaStream_t st,
                            const float* xtrue = nullptr, double* mpart = nullptr, double* metrics = nullptr);
size_t conv3_r4_metrics_part_bytes(int batch, int n1, int n2, int num_sms);
int conv3_tc_box_cols(int n2);
int conv3_tc_box_ch(bool tf32);
cudaError_t launch_conv3_tc(const CUtensorMap* tmH2, const void* w3pack, const float* bias, int fullmap, int relu,
                            float* xhat, int batch, int n1, int n2, int num_sms, bool tf32, cudaStream_t st);

// sensing model and metrics (k_sense.cu)
cudaError_t launch_stage_x(const float* x, int N, int ldo, int batch, void* out, bool bf16, cudaStream_t st);
cudaError_t launch_untranspose(const void* phiT, int m, int N, int kpad, int tr, int ldp, void* phi, bool bf16,
                               cudaStream_t st);
cudaError_t launch_measure_f32(const float* x, const float* phi, int m, int N, int batch, float* y, long long ldy,
                               cudaStream_t st);
cudaError_t launch_add_noise(void* y, long long ldy, int m, int batch, double snr_db, uint64_t key, bool bf16,
                             cudaStream_t st);
cudaError_t launch_metrics(const float* xhat, const float* x, int N, int batch, double* out, cudaStream_t st);

// training step, fp32 contexts (k_train.cu, k_conv_simt.cu)
constexpr int WGRAD_CHUNKS = 592;           // pixel-tile chunks of the weight-gradient reductions (4 x 148)
constexpr int N_PARAMS = 64 * 121 + 32 * 64 * 121 + 32 * 121 + 64 + 32 + 1;   // 259 521
cudaError_t launch_loss_grad(const float* xhat, const float* x, int N, int batch, double scale, float* dxhat,
                             double* loss_img, double* loss, cudaStream_t st);
cudaError_t launch_dgrad_mask(float* d, const float* y, size_t n, cudaStream_t st);
cudaError_t launch_dgrad3_f32(const float* dxhat, const float* wt3, const float* h2, float* dh2, int batch, int n1,
                              int n2, cudaStream_t st);
cudaError_t launch_dgrad2_f32(const float* dh2, const float* wt2, const float* h1, float* dh1, int batch, int n1,
                              int n2, cudaStream_t st);
cudaError_t launch_wgrad(int layer, const float* X, const float* dG, int batch, int n1, int n2, float* part_w,
                         float* part_b, int flip, float* gw, float* gb, cudaStream_t st);
cudaError_t launch_repack_tf32(const float* params, int flip, float* wp1, float* wp2t, float* wp3, float* wpd3,
                               void* wp2db, cudaStream_t st);
cudaError_t launch_repack_bf16(const float* params, int flip, void* wp1, void* wp2, void* wp3, cudaStream_t st);
cudaError_t launch_dgrad2_bf16(const CUtensorMap* tmDGb, const void* wpack, const void* h1b, int batch, int n1, int n2,
                               void* dh1b, int num_sms, cudaStream_t st);
// training: layer-2 data gradient on the bf16 layer-2 kernel (k_conv2_tc.cu); wpack = 66 blocks of 8 KB
constexpr int DG2_KBLOCKS = 66;
// training, TF32 contexts: layer-3 data gradient as a 1 -> 32 TF32 conv on the conv1 machinery (k_conv13_tc.cu);
// tmDX: the conv1 x_tilde tensor map over dG3; wpack: 11 x 4096 B (conv1 TF32 layout)
// custom stacks (NEXT-3): first layer 1 -> cout (32 or 64) in TF32 on the conv1 machinery (bank rows >= cout zero)
cudaError_t launch_conv1g_tf32(int cout, const CUtensorMap* tmX, const void* w1pack, const float* bias, float* out,
                               int batch, int n1, int n2, int num_sms, cudaStream_t st);
// custom stacks, FP32 SIMT: (cin, cout) in {(1,32), (1,64), (32,32), (32,64), (64,32), (64,64)}, bias + ReLU
cudaError_t launch_convg_simt(int cin, int cout, const float* in, const float* wx, const float* bias, float* out,
                              int batch, int n1, int n2, cudaStream_t st);
// training: dG2 = [h2 > 0] * (layer-3 dgrad of dG3) in bf16 + the layer-2 bias gradient (k_conv1_tf32<32, true>)
cudaError_t launch_dgrad3_tf32(const CUtensorMap* tmDX, const void* wpack, const void* h2, void* dg2b, float* part_b,
                               float* gb2, int batch, int n1, int n2, int num_sms, cudaStream_t st, bool h2_bf16);
// training, TF32 contexts: layer-2 weight gradient on tcgen05 from bf16 copies of h1 / dG2 (k_wgrad2_tc.cu)
constexpr int WG2_ROWS = 6;
size_t wgrad2_tc_smem_bytes(int n2);
int wgrad2_tc_h_box_rows();
int wgrad2_tc_g_box_rows();
size_t wgrad2_tc_part_floats(int num_sms);
cudaError_t setup_wgrad2_tc(int n2);
cudaError_t launch_wgrad2_tc(const CUtensorMap* tmH, const CUtensorMap* tmG, int batch, int n1, int n2, float* part,
                             int flip, float* gw, int num_sms, cudaStream_t st);
cudaError_t launch_to_bf16(const float* src, void* dst, size_t n, cudaStream_t st);
cudaError_t launch_dg2_bf16(const float* dg, size_t npix, void* dst, float* part_b, cudaStream_t st);
// training, TF32 contexts: layer-1 / layer-3 weight gradients on tcgen05 (k_wgrad13_tc.cu)
constexpr int WG13_ROWS = 6;
size_t wgrad13_tc_part_floats(int num_sms);
cudaError_t setup_wgrad13_tc(int n2);
// dg1: [B][N][64] bf16 (the bf16 dgrad2 output)
// xt / h2: fp32, or bf16 when xt_bf16 / h2_bf16 (BF16 contexts)
cudaError_t launch_wgrad1_tc(const void* xt, const void* dg1, int batch, int n1, int n2, float* part, float* part_b,
                             int flip, float* gw, float* gb, int num_sms, cudaStream_t st, bool xt_bf16 = false,
                             const CUtensorMap* tmD1 = nullptr);
int wgrad1_tc_d_box_rows();   // bf16 dG1 strip box of k_wgrad1_tc (64 ch x P x rows, SWIZZLE_128B)
cudaError_t launch_wgrad3_tc(const void* h2, const float* dg3, int batch, int n1, int n2, float* part, float* part_b,
                             int flip, float* gw, float* gb, int num_sms, cudaStream_t st, bool h2_bf16 = false,
                             const CUtensorMap* tmH2 = nullptr);
int wgrad3_tc_h_box_rows();   // bf16 h2 strip box of k_wgrad3_tc (32 ch x P x rows, SWIZZLE_64B)
cudaError_t launch_bias_reduce(const float* part_b, int nchunk, int nb, float* gb, cudaStream_t st);
// custom stacks (NEXT-3): generic SIMT weight / data gradients per layer, the per-layer repack, SGD, bf16 -> fp32
cudaError_t launch_wgrad_layer(int cin, int cout, const float* X, const float* dG, int batch, int n1, int n2,
                               float* part_w, float* part_b, int flip, float* gw, float* gb, cudaStream_t st);
size_t wgrad_layer_part_floats(int cin, int cout);
size_t wgrad_layer_partb_floats(int cin, int cout);
cudaError_t launch_dgrad_simt(int cin, int cout, const float* dG, const float* wt, const float* X, float* dX, int batch,
                              int n1, int n2, cudaStream_t st);
cudaError_t launch_repack_layer(const float* W, const float* b, int cin, int cout, int flip, float* wx, float* wt,
                                float* bdst, cudaStream_t st);
cudaError_t launch_sgd(float* params, const float* grads, float* vel, int n, float lr, float momentum, cudaStream_t st);
cudaError_t launch_bf16_to_f32(const void* src, int pitch, int ch, size_t npix, float* dst, cudaStream_t st);
cudaError_t launch_sgd_repack(float* params, const float* grads, float* vel, int n, float lr, float momentum, int flip,
                              float* wx1, float* wx2, float* wx3, float* wt2, float* wt3, float* b1, float* b2,
                              float* b3, cudaStream_t st);

}  // namespace di
