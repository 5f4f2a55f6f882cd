// k_train.cu -- the training step of DeepInverse for fp32 contexts:
//   loss      L = scale * sum_b ||x_hat_b - x_b||^2                       (scale = 1/l)
//   gradient  reverse-mode through the three conv layers of Eq. (1); the lifting layer
//             Phi^T is fixed and receives none
//   update    plain SGD with optional momentum ("backpropagation"; the optimiser is unstated)
// In the kernels' cross-correlation orientation (wx[co][ci][a][b], 'same' zero padding), with dG = dY * ReLU'(Y):
//   db[co]             = sum_{b,p} dG[p][co]
//   dwx[co][ci][a][b]  = sum_{b,p} dG[p][co] * X[p + (a-5, b-5)][ci]        (k_wgrad, this file)
//   dX[p][ci]          = sum_{co,a,b} wx[co][ci][10-a][10-b] dG[p + (a-5, b-5)][co]   (k_conv_wide with transposed,
//                        flipped weights and the previous activation as mask: k_conv_simt.cu)
// Reductions over pixels are two-level and deterministic: fp32 per block over its pixel tiles, then fp64 over
// blocks in a fixed order (k_wgrad_reduce).
#include <algorithm>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace di {

namespace {
constexpr int TH = 8, TW = 32;       // pixel tile
constexpr int KS = 11;
}  // namespace

// ----------------------------------------------------------------------------- loss and dL/dx_hat
// one block per image: dxhat = 2 scale (xhat - x); per-image loss partial (fp64) to loss_img[b]
__global__ void __launch_bounds__(256) k_loss_grad(const float* __restrict__ xhat, const float* __restrict__ x, int N,
                                                   double scale, float* __restrict__ dxhat,
                                                   double* __restrict__ loss_img) {
  __shared__ double red[8];
  const size_t off = (size_t)blockIdx.x * N;
  double acc = 0.0;
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    const float d = xhat[off + j] - x[off + j];
    acc += (double)d * d;
    dxhat[off + j] = (float)(2.0 * scale) * d;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    loss_img[blockIdx.x] = scale * t;
  }
}

// dG3 = dx_hat * 1(x_hat > 0) when the last layer applies ReLU (DI_FLAG_FINAL_RELU)
__global__ void k_mask(float* __restrict__ d, const float* __restrict__ y, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    if (!(y[i] > 0.f)) d[i] = 0.f;
}
cudaError_t launch_dgrad_mask(float* d, const float* y, size_t n, cudaStream_t st) {
  k_mask<<<1184, 256, 0, st>>>(d, y, n);
  return cudaGetLastError();
}

// sum of per-image losses -> loss[0]: lane l sums images l, l + 32, ... then a fixed butterfly (deterministic)
__global__ void k_sum_f64(const double* __restrict__ v, int n, double* __restrict__ out) {
  double t = 0.0;
  for (int i = threadIdx.x; i < n; i += 32) t += v[i];
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (threadIdx.x == 0) *out = t;
}

cudaError_t launch_loss_grad(const float* xhat, const float* x, int N, int batch, double scale, float* dxhat,
                             double* loss_img, double* loss, cudaStream_t st) {
  k_loss_grad<<<batch, 256, 0, st>>>(xhat, x, N, scale, dxhat, loss_img);
  k_sum_f64<<<1, 32, 0, st>>>(loss_img, batch, loss);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- weight gradients
// Block (ci-chunk, co-chunk) x pixel-tile chunk; thread (co_l, ci_l, ag) accumulates the taps (a, b) with
// a = ag, ag + 4, ag + 8 (< 11) and all 11 b for its (co, ci) over the block's pixel tiles: per tap row a and pixel
// row r, one 42-wide X row in registers slides under the 32 dG values of that row (352 FMAs per 74 loads).
// Threads with ci_l = 0, ag = 0 of the ci-chunk-0 blocks also sum dG for the bias gradient.
template <int CIN, int COUT, int CI_T, int CO_T>
__global__ void __launch_bounds__(CI_T * CO_T * 4)
    k_wgrad(const float* __restrict__ X, const float* __restrict__ dG, int batch, int n1, int n2, int nchunk,
            float* __restrict__ part_w, float* __restrict__ part_b) {
  constexpr int NT = CI_T * CO_T * 4;
  constexpr int HT = TH + 10, WT = TW + 10;
  __shared__ float sx[CI_T][HT][WT];
  __shared__ float sg[CO_T][TH][TW];
  const int ci0 = (blockIdx.x % (CIN / CI_T)) * CI_T, co0 = (blockIdx.x / (CIN / CI_T)) * CO_T;
  const int chunk = blockIdx.y;
  const int tid = threadIdx.x;
  const int ag = tid / (CI_T * CO_T), rem = tid % (CI_T * CO_T);
  const int co_l = rem / CI_T, ci_l = rem % CI_T;
  const bool do_bias = ci0 == 0 && ci_l == 0 && ag == 0;
  float acc[3][KS];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < KS; ++j) acc[i][j] = 0.f;
  float bacc = 0.f;
  const int tx = (n2 + TW - 1) / TW, ty = (n1 + TH - 1) / TH;
  const long long ntiles = (long long)batch * tx * ty;
  for (long long t = chunk; t < ntiles; t += nchunk) {
    const int b = (int)(t / (tx * ty)), tr = (int)(t % (tx * ty));
    const int y0 = (tr / tx) * TH, x0 = (tr % tx) * TW;
    __syncthreads();
    for (int e = tid; e < CI_T * HT * WT; e += NT) {
      const int c = e / (HT * WT), r2 = e % (HT * WT), yy = r2 / WT, xx = r2 % WT;
      const int gy = y0 + yy - 5, gx = x0 + xx - 5;
      sx[c][yy][xx] = (gy >= 0 && gy < n1 && gx >= 0 && gx < n2)
                          ? X[(((size_t)b * n1 + gy) * n2 + gx) * CIN + ci0 + c] : 0.f;
    }
    for (int e = tid; e < CO_T * TH * TW; e += NT) {
      const int c = e / (TH * TW), r2 = e % (TH * TW), yy = r2 / TW, xx = r2 % TW;
      const int gy = y0 + yy, gx = x0 + xx;
      sg[c][yy][xx] = (gy < n1 && gx < n2) ? dG[(((size_t)b * n1 + gy) * n2 + gx) * COUT + co0 + c] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int ai = 0; ai < 3; ++ai) {
      const int a = ag + 4 * ai;
      if (a >= KS) continue;
#pragma unroll 1
      for (int r = 0; r < TH; ++r) {
        float xr[WT];
#pragma unroll
        for (int j = 0; j < WT; ++j) xr[j] = sx[ci_l][r + a][j];
#pragma unroll
        for (int px = 0; px < TW; ++px) {
          const float g = sg[co_l][r][px];
#pragma unroll
          for (int bb = 0; bb < KS; ++bb) acc[ai][bb] = fmaf(g, xr[px + bb], acc[ai][bb]);
        }
      }
    }
    if (do_bias)
      for (int i = 0; i < TH * TW; ++i) bacc += sg[co_l][i / TW][i % TW];
  }
  // partial[chunk][co][ci][a][b]
  float* pw = part_w + (size_t)chunk * COUT * CIN * KS * KS;
#pragma unroll
  for (int ai = 0; ai < 3; ++ai) {
    const int a = ag + 4 * ai;
    if (a >= KS) continue;
#pragma unroll
    for (int bb = 0; bb < KS; ++bb)
      pw[(((size_t)(co0 + co_l) * CIN + ci0 + ci_l) * KS + a) * KS + bb] = acc[ai][bb];
  }
  if (do_bias) part_b[(size_t)chunk * COUT + co0 + co_l] = bacc;
}

// As k_wgrad for an even number of output channels per block, with packed FFMA2 (fma.rn.f32x2: two IEEE fp32 FMAs,
// bit-identical to fmaf): a thread owns the channel PAIR (co, co + 1) of one ci, the pair's dG values sit side by
// side in shared memory (one LDS.64), the sliding X value is broadcast into the operand -- half the FMA
// instructions of two k_wgrad threads.
__device__ __forceinline__ void ffma2_t(uint64_t& d, float a, uint64_t b) {   // d = (a, a) * b + d per half, RN
  uint64_t aa;
  asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(aa), "l"(b));
}
template <int CIN, int COUT, int CI_T, int CO_T>
__global__ void __launch_bounds__(CI_T * CO_T * 2)
    k_wgrad_pair(const float* __restrict__ X, const float* __restrict__ dG, int batch, int n1, int n2, int nchunk,
                 float* __restrict__ part_w, float* __restrict__ part_b) {
  constexpr int NP = CO_T / 2;                       // channel pairs per block
  constexpr int NT = CI_T * NP * 4;
  constexpr int HT = TH + 10, WT = TW + 10;
  __shared__ float sx[CI_T][HT][WT];
  __shared__ __align__(8) float sg[NP][TH][TW][2];   // (co, co + 1) interleaved
  const int ci0 = (blockIdx.x % (CIN / CI_T)) * CI_T, co0 = (blockIdx.x / (CIN / CI_T)) * CO_T;
  const int chunk = blockIdx.y;
  const int tid = threadIdx.x;
  const int ag = tid / (CI_T * NP), rem = tid % (CI_T * NP);
  const int cp = rem / CI_T, ci_l = rem % CI_T;
  const bool do_bias = ci0 == 0 && ci_l == 0 && ag == 0;
  uint64_t acc[3][KS];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < KS; ++j) acc[i][j] = 0ull;
  float bacc0 = 0.f, bacc1 = 0.f;
  const int tx = (n2 + TW - 1) / TW, ty = (n1 + TH - 1) / TH;
  const long long ntiles = (long long)batch * tx * ty;
  for (long long t = chunk; t < ntiles; t += nchunk) {
    const int b = (int)(t / (tx * ty)), tr = (int)(t % (tx * ty));
    const int y0 = (tr / tx) * TH, x0 = (tr % tx) * TW;
    __syncthreads();
    for (int e = tid; e < CI_T * HT * WT; e += NT) {
      const int c = e / (HT * WT), r2 = e % (HT * WT), yy = r2 / WT, xx = r2 % WT;
      const int gy = y0 + yy - 5, gx = x0 + xx - 5;
      sx[c][yy][xx] = (gy >= 0 && gy < n1 && gx >= 0 && gx < n2)
                          ? X[(((size_t)b * n1 + gy) * n2 + gx) * CIN + ci0 + c] : 0.f;
    }
    for (int e = tid; e < CO_T * TH * TW; e += NT) {
      const int c = e % CO_T, pix = e / CO_T, yy = pix / TW, xx = pix % TW;   // channel innermost: coalesced
      const int gy = y0 + yy, gx = x0 + xx;
      sg[c >> 1][yy][xx][c & 1] = (gy < n1 && gx < n2) ? dG[(((size_t)b * n1 + gy) * n2 + gx) * COUT + co0 + c] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int ai = 0; ai < 3; ++ai) {
      const int a = ag + 4 * ai;
      if (a >= KS) continue;
#pragma unroll 1
      for (int r = 0; r < TH; ++r) {
        float xr[WT];
#pragma unroll
        for (int j = 0; j < WT; ++j) xr[j] = sx[ci_l][r + a][j];
#pragma unroll
        for (int px = 0; px < TW; ++px) {
          const uint64_t g = *reinterpret_cast<const uint64_t*>(&sg[cp][r][px][0]);
#pragma unroll
          for (int bb = 0; bb < KS; ++bb) ffma2_t(acc[ai][bb], xr[px + bb], g);
        }
      }
    }
    if (do_bias)
      for (int i = 0; i < TH * TW; ++i) bacc0 += sg[cp][i / TW][i % TW][0], bacc1 += sg[cp][i / TW][i % TW][1];
  }
  float* pw = part_w + (size_t)chunk * COUT * CIN * KS * KS;
  const int co = co0 + 2 * cp;
#pragma unroll
  for (int ai = 0; ai < 3; ++ai) {
    const int a = ag + 4 * ai;
    if (a >= KS) continue;
#pragma unroll
    for (int bb = 0; bb < KS; ++bb) {
      float lo, hi;
      asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[ai][bb]));
      pw[(((size_t)co * CIN + ci0 + ci_l) * KS + a) * KS + bb] = lo;
      pw[(((size_t)(co + 1) * CIN + ci0 + ci_l) * KS + a) * KS + bb] = hi;
    }
  }
  if (do_bias) part_b[(size_t)chunk * COUT + co] = bacc0, part_b[(size_t)chunk * COUT + co + 1] = bacc1;
}

// dW (API orientation) = sum over chunks (fp64, chunk order); xcorr-orientation tap (a, b) is the user's (u, v) =
// (10 - a, 10 - b) unless the context was created with DI_FLAG_XCORR
__global__ void k_wgrad_reduce(const float* __restrict__ part_w, const float* __restrict__ part_b, int nchunk,
                               int nw, int nb, int flip, float* __restrict__ gw, float* __restrict__ gb) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nw + nb; i += gridDim.x * blockDim.x) {
    double t = 0.0;
    if (i < nw) {
      for (int c = 0; c < nchunk; ++c) t += part_w[(size_t)c * nw + i];
      const int tap = i % (KS * KS), base = i - tap, a = tap / KS, b = tap % KS;
      gw[base + (flip ? (KS - 1 - a) * KS + (KS - 1 - b) : tap)] = (float)t;
    } else {
      const int j = i - nw;
      for (int c = 0; c < nchunk; ++c) t += part_b[(size_t)c * nb + j];
      gb[j] = (float)t;
    }
  }
}

template <int CIN, int COUT, int CI_T, int CO_T>
static cudaError_t wgrad(const float* X, const float* dG, int batch, int n1, int n2, int nchunk, float* part_w,
                         float* part_b, int flip, float* gw, float* gb, cudaStream_t st) {
  dim3 grid((CIN / CI_T) * (COUT / CO_T), nchunk);
  if constexpr (CO_T % 2 == 0)
    k_wgrad_pair<CIN, COUT, CI_T, CO_T><<<grid, CI_T * CO_T * 2, 0, st>>>(X, dG, batch, n1, n2, nchunk, part_w,
                                                                         part_b);
  else
    k_wgrad<CIN, COUT, CI_T, CO_T><<<grid, CI_T * CO_T * 4, 0, st>>>(X, dG, batch, n1, n2, nchunk, part_w, part_b);
  const int nw = COUT * CIN * KS * KS;
  k_wgrad_reduce<<<(nw + COUT + 255) / 256, 256, 0, st>>>(part_w, part_b, nchunk, nw, COUT, flip, gw, gb);
  return cudaGetLastError();
}

// gb[j] = sum over chunks of part_b[chunk][j]: one block per output, fixed strided fp64 partials + fixed tree
__global__ void __launch_bounds__(256) k_bias_reduce(const float* __restrict__ part_b, int nchunk, int nb,
                                                     float* __restrict__ gb) {
  __shared__ double sh[256];
  const int j = blockIdx.x;
  double t = 0.0;
  for (int c = threadIdx.x; c < nchunk; c += 256) t += part_b[(size_t)c * nb + j];
  sh[threadIdx.x] = t;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) gb[j] = (float)sh[0];
}

cudaError_t launch_bias_reduce(const float* part_b, int nchunk, int nb, float* gb, cudaStream_t st) {
  k_bias_reduce<<<nb, 256, 0, st>>>(part_b, nchunk, nb, gb);
  return cudaGetLastError();
}

// layer 3: X = h2 (32 ch), dG = dx_hat (1 ch); layer 2: X = h1 (64), dG = dh2 (32); layer 1: X = x_tilde (1),
// dG = dh1 (64).  part_w / part_b: scratch of WGRAD_CHUNKS x (weights / biases of the layer).
cudaError_t launch_wgrad(int layer, const float* X, const float* dG, int batch, int n1, int n2, float* part_w,
                         float* part_b, int flip, float* gw, float* gb, cudaStream_t st) {
  // (CI_T, CO_T) keep the static tiles under 48 KB; grid.x * nchunk ~ WGRAD_CHUNKS blocks
  switch (layer) {
    case 3: return wgrad<32, 1, 8, 1>(X, dG, batch, n1, n2, WGRAD_CHUNKS / 4, part_w, part_b, flip, gw, gb, st);
    case 2: return wgrad<64, 32, 8, 8>(X, dG, batch, n1, n2, WGRAD_CHUNKS / 32, part_w, part_b, flip, gw, gb, st);
    default: return wgrad<1, 64, 1, 16>(X, dG, batch, n1, n2, WGRAD_CHUNKS / 4, part_w, part_b, flip, gw, gb, st);
  }
}

// ----------------------------------------------------------------------------- custom stacks (NEXT-3)
// Weight gradient of one layer of a custom stack, any (C_in, C_out) a stack may hold:
// the same register-blocked sliding-window kernels as the paper's layers, instantiated per channel pair.
static int wgrad_layer_chunks(int cin, int cout) {   // WGRAD_CHUNKS / (blocks per chunk of the instance below)
  if (cin == 1) return WGRAD_CHUNKS / (cout == 32 ? 2 : 4);
  if (cout == 1) return WGRAD_CHUNKS / 4;
  return std::max(1, WGRAD_CHUNKS / ((cin / 8) * (cout / 8)));
}
cudaError_t launch_wgrad_layer(int cin, int cout, const float* X, const float* dG, int batch, int n1, int n2,
                               float* part_w, float* part_b, int flip, float* gw, float* gb, cudaStream_t st) {
  const int C = wgrad_layer_chunks(cin, cout);
  if (cin == 1 && cout == 32) return wgrad<1, 32, 1, 16>(X, dG, batch, n1, n2, C, part_w, part_b, flip, gw, gb, st);
  if (cin == 1 && cout == 64) return wgrad<1, 64, 1, 16>(X, dG, batch, n1, n2, C, part_w, part_b, flip, gw, gb, st);
  if (cin == 32 && cout == 32) return wgrad<32, 32, 8, 8>(X, dG, batch, n1, n2, C, part_w, part_b, flip, gw, gb, st);
  if (cin == 32 && cout == 64) return wgrad<32, 64, 8, 8>(X, dG, batch, n1, n2, C, part_w, part_b, flip, gw, gb, st);
  if (cin == 64 && cout == 32) return wgrad<64, 32, 8, 8>(X, dG, batch, n1, n2, C, part_w, part_b, flip, gw, gb, st);
  if (cin == 64 && cout == 64) return wgrad<64, 64, 8, 8>(X, dG, batch, n1, n2, C, part_w, part_b, flip, gw, gb, st);
  if (cin == 32 && cout == 1) return wgrad<32, 1, 8, 1>(X, dG, batch, n1, n2, C, part_w, part_b, flip, gw, gb, st);
  if (cin == 32 && cout == 128) return wgrad<32, 128, 8, 8>(X, dG, batch, n1, n2, C, part_w, part_b, flip, gw, gb, st);
  if (cin == 64 && cout == 128) return wgrad<64, 128, 8, 8>(X, dG, batch, n1, n2, C, part_w, part_b, flip, gw, gb, st);
  if (cin == 128 && cout == 128) return wgrad<128, 128, 8, 8>(X, dG, batch, n1, n2, C, part_w, part_b, flip, gw, gb, st);
  if (cin == 128 && cout == 64) return wgrad<128, 64, 8, 8>(X, dG, batch, n1, n2, C, part_w, part_b, flip, gw, gb, st);
  if (cin == 128 && cout == 32) return wgrad<128, 32, 8, 8>(X, dG, batch, n1, n2, C, part_w, part_b, flip, gw, gb, st);
  return cudaErrorInvalidValue;
}
// scratch floats launch_wgrad_layer needs: part_w (chunks x weights of the layer); part_b needs chunks x cout
size_t wgrad_layer_part_floats(int cin, int cout) {
  return (size_t)wgrad_layer_chunks(cin, cout) * cin * cout * KS * KS;
}
size_t wgrad_layer_partb_floats(int cin, int cout) { return (size_t)wgrad_layer_chunks(cin, cout) * cout; }

// From the API-orientation parameters of one layer (W [cout][cin][11][11], b [cout]): the forward SIMT layout
// wx[ci][a][b][co] of the cross-correlation taps (FP32 contexts; may be null), the backward layout
// wt[co][10-a][10-b][ci] (the data gradient is a 'same' correlation of dG with the rotated, transposed bank) and the
// bias array (may be null)
__global__ void k_repack_layer(const float* __restrict__ W, const float* __restrict__ bsrc, int cin, int cout, int flip,
                               float* __restrict__ wx, float* __restrict__ wt, float* __restrict__ bdst) {
  const int nw = cout * cin * KS * KS;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nw + cout; i += gridDim.x * blockDim.x) {
    if (i >= nw) {
      if (bdst) bdst[i - nw] = bsrc[i - nw];
      continue;
    }
    const int tap = i % (KS * KS), co = i / (KS * KS) / cin, ci = (i / (KS * KS)) % cin;
    const int u = tap / KS, v = tap % KS;
    const int a = flip ? KS - 1 - u : u, b = flip ? KS - 1 - v : v;
    const float w = W[i];
    if (wx) wx[(((size_t)ci * KS + a) * KS + b) * cout + co] = w;
    if (wt) wt[(((size_t)co * KS + (KS - 1 - a)) * KS + (KS - 1 - b)) * cin + ci] = w;
  }
}
cudaError_t launch_repack_layer(const float* W, const float* b, int cin, int cout, int flip, float* wx, float* wt,
                                float* bdst, cudaStream_t st) {
  const int n = cout * cin * KS * KS + cout;
  k_repack_layer<<<(n + 255) / 256 < 592 ? (n + 255) / 256 : 592, 256, 0, st>>>(W, b, cin, cout, flip, wx, wt, bdst);
  return cudaGetLastError();
}

// bf16 activation [npix][pitch] -> fp32 [npix][ch] (the custom stack's training forward keeps every layer's output)
__global__ void k_bf16_to_f32(const __nv_bfloat16* __restrict__ src, int pitch, int ch, size_t npix,
                              float* __restrict__ dst) {
  const size_t n = npix * ch;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t p = i / ch;
    dst[i] = __bfloat162float(src[p * pitch + (i - p * ch)]);
  }
}
cudaError_t launch_bf16_to_f32(const void* src, int pitch, int ch, size_t npix, float* dst, cudaStream_t st) {
  k_bf16_to_f32<<<1184, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(src), pitch, ch, npix, dst);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- SGD and weight repacking
// params / grads / vel: [W1 (64*121) | W2 (32*64*121) | W3 (32*121) | b1 (64) | b2 (32) | b3 (1)] in the API
// orientation.  vel = momentum * vel + grad; param -= lr * vel.
__global__ void k_sgd(float* __restrict__ params, const float* __restrict__ grads, float* __restrict__ vel, int n,
                      float lr, float momentum) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float v = momentum * vel[i] + grads[i];
    vel[i] = v;
    params[i] -= lr * v;
  }
}

// from the API-orientation parameters: the forward SIMT layouts wx_l[ci][a][b][co] (cross-correlation taps), the
// backward layouts wt3[0][a][b][c] = wx3[0][c][10-a][10-b] and wt2[k][a][b][c] = wx2[k][c][10-a][10-b] (co <-> ci
// swapped), and the per-channel bias arrays
__global__ void k_repack(const float* __restrict__ params, int flip, float* __restrict__ wx1, float* __restrict__ wx2,
                         float* __restrict__ wx3, float* __restrict__ wt2, float* __restrict__ wt3,
                         float* __restrict__ b1, float* __restrict__ b2, float* __restrict__ b3) {
  constexpr int T = KS * KS, N1 = 64 * T, N2 = 32 * 64 * T, N3 = 32 * T;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N1 + N2 + N3 + 97; i += gridDim.x * blockDim.x) {
    if (i >= N1 + N2 + N3) {
      const int j = i - (N1 + N2 + N3);
      const float v = params[i];
      if (j < 64) b1[j] = v; else if (j < 96) b2[j - 64] = v; else b3[0] = v;
      continue;
    }
    int li, co, ci, cin, cout;
    if (i < N1) li = i, cin = 1, cout = 64;
    else if (i < N1 + N2) li = i - N1, cin = 64, cout = 32;
    else li = i - N1 - N2, cin = 32, cout = 1;
    const int tap = li % T;
    co = li / T / cin, ci = (li / T) % cin;
    const int u = tap / KS, v = tap % KS;
    const int a = flip ? KS - 1 - u : u, b = flip ? KS - 1 - v : v;     // cross-correlation tap (a, b)
    const float w = params[i];
    const size_t fwd = (((size_t)ci * KS + a) * KS + b) * cout + co;    // [ci][a][b][co]
    if (i < N1) {
      wx1[fwd] = w;
    } else if (i < N1 + N2) {
      wx2[fwd] = w;
      wt2[(((size_t)co * KS + (KS - 1 - a)) * KS + (KS - 1 - b)) * 64 + ci] = w;   // [k=co][a'][b'][c=ci]
    } else {
      wx3[fwd] = w;
      wt3[(((size_t)0 * KS + (KS - 1 - a)) * KS + (KS - 1 - b)) * 32 + ci] = w;    // [0][a'][b'][c=ci]
    }
  }
}

// TF32 contexts: the tensor-core weight images (k_conv13_tc.cu / k_conv2_tf32.cu layouts, same as api.cu's host
// packers) re-derived on the device from the parameters after every SGD step
__device__ __forceinline__ float wx_at(const float* __restrict__ W, int cin, int co, int ci, int a, int b, int flip) {
  const int u = flip ? KS - 1 - a : a, v = flip ? KS - 1 - b : b;
  return W[(((size_t)co * cin + ci) * KS + u) * KS + v];
}

__global__ void k_repack_tf32(const float* __restrict__ params, int flip, float* __restrict__ wp1,
                              float* __restrict__ wp2t, float* __restrict__ wp3, float* __restrict__ wpd3,
                              uint16_t* __restrict__ wp2db) {
  constexpr int T = KS * KS, N1 = 64 * T, N2 = 32 * 64 * T;
  const float* W1 = params;
  const float* W2 = params + N1;
  const float* W3 = params + N1 + N2;
  constexpr int E2 = 2 * 33 * 4096, E1 = 11 * 1024, E3 = 22 * 512, E4 = 0, E5 = 11 * 1024;
  constexpr int E6 = DG2_KBLOCKS * 4096;   // bf16 layer-2 dgrad blocks: 66 x (128 rows x 32 co x 2 B), SWIZZLE_64B
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E2 + E1 + E3 + E4 + E5 + E6; e += gridDim.x * blockDim.x) {
    if (e >= E2 + E1 + E3 + E4 + E5) {
      if (!wp2db) continue;
      const int i = e - E2 - E1 - E3 - E4 - E5;
      const int blk = i / 4096, u = blk / 6, j = blk % 6, o = (i % 4096) * 2, row = o / 64, r = o % 64;
      const int co = (((r / 16) ^ ((row >> 1) & 3)) * 8) + (r % 16) / 2;
      const int bb = 2 * j + row / 64, ci = row % 64;
      const float v = bb < KS ? wx_at(W2, 64, co, ci, KS - 1 - u, KS - 1 - bb, flip) : 0.f;
      wp2db[i] = __bfloat16_as_ushort(__float2bfloat16_rn(v));
      continue;
    }
    if (e < E2) {                     // conv2: [h][kb] blocks of 128 rows x 32 ch, SWIZZLE_128B
      if (!wp2t) continue;
      const int blk = e / 4096, o = (e % 4096) * 4, row = o / 128, r = o % 128;
      const int c = (((r / 16) ^ (row & 7)) * 4) + (r % 16) / 4;
      const int h = blk / 33, kb = blk % 33, u = kb / 3, b = 4 * (kb % 3) + row / 32, k = row % 32;
      wp2t[e] = b < KS ? wx_at(W2, 64, k, 32 * h + c, u, b, flip) : 0.f;
    } else if (e < E2 + E1) {         // conv1: [u] blocks of 64 permuted filters x 16 taps, SWIZZLE_64B
      if (!wp1) continue;
      const int i = e - E2, u = i / 1024, o = (i % 1024) * 4, m = o / 64, r = o % 64;
      const int v = (((r / 16) ^ ((m >> 1) & 3)) * 4) + (r % 16) / 4;
      const int grp = m / 16, j = m % 16, f = 16 * grp + (j < 8 ? 2 * j : 2 * (j - 8) + 1);
      wp1[i] = v < KS ? wx_at(W1, 1, f, 0, u, v, flip) : 0.f;
    } else if (e < E2 + E1 + E3) {    // conv3: [h*11 + u] blocks of 32 rows (taps v) x 16 ch, SWIZZLE_64B
      if (!wp3) continue;
      const int i = e - E2 - E1, blk = i / 512, h = blk / 11, u = blk % 11, o = (i % 512) * 4, row = o / 64,
                r = o % 64;
      const int c = (((r / 16) ^ ((row >> 1) & 3)) * 4) + (r % 16) / 4;
      wp3[i] = row < KS ? wx_at(W3, 32, 0, 16 * h + c, u, row, flip) : 0.f;
    } else if (e >= E2 + E1 + E3 + E4) {   // layer-3 dgrad as a conv1-layout bank: filter f < 32 = ci, rotated taps
      if (!wpd3) continue;
      const int i = e - E2 - E1 - E3 - E4, u = i / 1024, o = (i % 1024) * 4, m = o / 64, r = o % 64;
      const int v = (((r / 16) ^ ((m >> 1) & 3)) * 4) + (r % 16) / 4;
      const int grp = m / 16, j = m % 16, f = 16 * grp + (j < 8 ? 2 * j : 2 * (j - 8) + 1);
      wpd3[i] = (v < KS && f < 32) ? wx_at(W3, 32, 0, f, KS - 1 - u, KS - 1 - v, flip) : 0.f;
    }
  }
}

// BF16 contexts: the bf16 forward images (api.cu conv1_tc_pack / conv2_tc_pack / conv3_r4_pack), RNE-rounded
__device__ __forceinline__ uint16_t bfbits(float v) { return __bfloat16_as_ushort(__float2bfloat16_rn(v)); }

__global__ void k_repack_bf16(const float* __restrict__ params, int flip, uint16_t* __restrict__ wp1,
                              uint16_t* __restrict__ wp2, uint16_t* __restrict__ wp3) {
  constexpr int T = KS * KS, N1 = 64 * T, N2 = 32 * 64 * T;
  const float* W1 = params;
  const float* W2 = params + N1;
  const float* W3 = params + N1 + N2;
  constexpr int E2 = 33 * 8192, E1 = 11 * 1024, E3 = C3R_NENT * C3R_ES * 32;   // bf16 elements per image
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E2 + E1 + E3; e += gridDim.x * blockDim.x) {
    if (e < E2) {                     // conv2: block u*3 + j, row v'*32 + k, 64 ci (128 B), SWIZZLE_128B
      const int kb = e / 8192, o = (e % 8192) * 2, row = o / 128, r = o % 128;
      const int ci = (((r / 16) ^ (row & 7)) * 8) + (r % 16) / 2;
      const int u = kb / 3, b = 4 * (kb % 3) + row / 32, k = row % 32;
      wp2[e] = bfbits(b < KS ? wx_at(W2, 64, k, ci, u, b, flip) : 0.f);
    } else if (e < E2 + E1) {         // conv1: block u, row m (filter m), 16 taps (32 B), SWIZZLE_32B
      const int i = e - E2, u = i / 1024, o = (i % 1024) * 2, m = o / 32, r = o % 32;
      const int v = (((r / 16) ^ ((m >> 2) & 1)) * 8) + (r % 16) / 2;
      const int f = m;
      wp1[i] = bfbits(v < KS ? wx_at(W1, 1, f, 0, u, v, flip) : 0.f);
    } else {                          // conv3 (k_conv3_r4): stack row rho = entry e x ES + tap v, 32 ch, SW64
      const int i = e - E2 - E1, rho = i / 32, o = (i % 32) * 2;
      const int c = ((((o / 16) ^ ((rho >> 1) & 3))) * 8) + (o % 16) / 2;
      const int v = rho % C3R_ES, u = 10 - (rho / C3R_ES + C3R_IMIN);
      wp3[i] = bfbits((v < KS && u >= 0 && u < KS) ? wx_at(W3, 32, 0, c, u, v, flip) : 0.f);
    }
  }
}

cudaError_t launch_repack_bf16(const float* params, int flip, void* wp1, void* wp2, void* wp3, cudaStream_t st) {
  k_repack_bf16<<<592, 256, 0, st>>>(params, flip, reinterpret_cast<uint16_t*>(wp1), reinterpret_cast<uint16_t*>(wp2),
                                     reinterpret_cast<uint16_t*>(wp3));
  return cudaGetLastError();
}

cudaError_t launch_repack_tf32(const float* params, int flip, float* wp1, float* wp2t, float* wp3, float* wpd3,
                               void* wp2db, cudaStream_t st) {
  k_repack_tf32<<<592, 256, 0, st>>>(params, flip, wp1, wp2t, wp3, wpd3, reinterpret_cast<uint16_t*>(wp2db));
  return cudaGetLastError();
}

cudaError_t launch_sgd(float* params, const float* grads, float* vel, int n, float lr, float momentum, cudaStream_t st) {
  k_sgd<<<296, 256, 0, st>>>(params, grads, vel, n, lr, momentum);
  return cudaGetLastError();
}

cudaError_t launch_sgd_repack(float* params, const float* grads, float* vel, int n, float lr, float momentum, int flip,
                              float* wx1, float* wx2, float* wx3, float* wt2, float* wt3, float* b1, float* b2,
                              float* b3, cudaStream_t st) {
  if (grads) k_sgd<<<296, 256, 0, st>>>(params, grads, vel, n, lr, momentum);
  k_repack<<<296, 256, 0, st>>>(params, flip, wx1, wx2, wx3, wt2, wt3, b1, b2, b3);
  return cudaGetLastError();
}

}  // namespace di
