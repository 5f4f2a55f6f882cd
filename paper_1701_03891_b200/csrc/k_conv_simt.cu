// k_conv_simt.cu -- SIMT (FFMA) convolution layers of Eq. (1):
//   * conv layer 1 (1 -> 64, ReLU) for all precisions,
//   * conv layer 2 (64 -> 32, ReLU) for the fp32 path,
//   * conv layer 3 (32 -> 1, optional ReLU) for all precisions.
// Each computes the 'same' zero-padded cross-correlation with the flipped taps (== full convolution
// followed by the centred crop S) in fp32 with two-level accumulation (per input
// channel over the 121 taps, then over channels), reading NHWC inputs through a shared-memory halo
// tile that is zero outside the image (the zero padding of Eq. (1)).
//
// Weight layout (packed by di_create): wx[ci][a][b][co] fp32, a,b in 0..10, xcorr orientation.
// Bias: per-channel b[co], or (fullmap) the cropped map bm[r][c][co].
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace di {

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

// packed fp32 pairs for FFMA2 (fma.rn.f32x2, sm_100a)
__device__ __forceinline__ uint64_t f32x2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ uint64_t f32x2_bcast(float x) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void f32x2_unpack(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ void ffma2(uint64_t& d, uint64_t a, uint64_t b) {   // d = a * b + d, per half, RN
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}

// ---------------------------------------------------------------------------------------------
// wide-output layers (C_out >= 16): block tile TH x TW pixels x all COUT channels; thread computes
// PX pixels (strided by TW/PX along x, conflict-free smem reads) x CO_T channels.
template <typename Tin, typename Tout, int CIN, int COUT, int CO_T, int CI_CHUNK>
__global__ void __launch_bounds__(256)
    k_conv_wide(const Tin* __restrict__ in, const float* __restrict__ wx, const float* __restrict__ bias, int fullmap,
                const Tout* __restrict__ mask,
                int relu, Tout* __restrict__ out, int n1, int n2) {
  constexpr int TH = 8, TW = 32, PX = 4;
  constexpr int HT = TH + 10, WT = TW + 10;
  constexpr int WTS = 72;   // smem row stride: 72 = 8 (mod 32), so the 4 rows x 8 columns a warp reads hit 32 banks
  constexpr int PIX_THREADS = TH * TW / PX;       // 64
  constexpr int CO_GROUPS = COUT / CO_T;
  static_assert(PIX_THREADS * CO_GROUPS == 256, "256 threads");
  extern __shared__ float sm[];
  float* sx = sm;                                  // [CI_CHUNK][HT][WTS]
  float* sw = sm + CI_CHUNK * HT * WTS;            // [CI_CHUNK][121][COUT]

  const int b = blockIdx.z;
  const int y0 = blockIdx.y * TH, x0 = blockIdx.x * TW;
  const int tid = threadIdx.x;
  const int cg = tid / PIX_THREADS, pt = tid % PIX_THREADS;
  const int py = pt / (TW / PX), pxb = pt % (TW / PX);   // pixel (py, pxb + p*(TW/PX))
  float acc[PX][CO_T];
#pragma unroll
  for (int p = 0; p < PX; ++p)
#pragma unroll
    for (int c = 0; c < CO_T; ++c) acc[p][c] = 0.f;

  for (int ci0 = 0; ci0 < CIN; ci0 += CI_CHUNK) {
    __syncthreads();
    for (int e = tid; e < CI_CHUNK * HT * WT; e += 256) {   // channel innermost: neighbouring threads, one pixel
      const int cc = e % CI_CHUNK, pix = e / CI_CHUNK;
      const int yy = pix / WT, xx = pix - yy * WT;
      const int gy = y0 + yy - 5, gx = x0 + xx - 5;
      float v = 0.f;
      if (gy >= 0 && gy < n1 && gx >= 0 && gx < n2)
        v = to_f(in[(((size_t)b * n1 + gy) * n2 + gx) * CIN + ci0 + cc]);
      sx[(cc * HT + yy) * WTS + xx] = v;
    }
    for (int e = tid; e < CI_CHUNK * 121 * COUT; e += 256) sw[e] = wx[(size_t)ci0 * 121 * COUT + e];
    __syncthreads();
#pragma unroll 1
    for (int cc = 0; cc < CI_CHUNK; ++cc) {
      // per-channel partial sums as packed fp32 pairs (channels c, c+1): one fma.rn.f32x2 (FFMA2, two IEEE fp32
      // FMAs -- bit-identical to fmaf) per pixel and channel pair, the pixel value broadcast by ptxas into the
      // operand: half the FMA instructions, so the loop is bound by the FMA pipe instead of instruction issue
      uint64_t part[PX][CO_T / 2];
#pragma unroll
      for (int p = 0; p < PX; ++p)
#pragma unroll
        for (int c = 0; c < CO_T / 2; ++c) part[p][c] = 0ull;
      const float* xr = sx + cc * HT * WTS + py * WTS + pxb;
      const float* wr = sw + cc * 121 * COUT + cg * CO_T;
#pragma unroll 1
      for (int a = 0; a < 11; ++a) {
#pragma unroll
        for (int bb = 0; bb < 11; ++bb) {
          uint64_t xv[PX];
#pragma unroll
          for (int p = 0; p < PX; ++p) xv[p] = f32x2_bcast(xr[a * WTS + bb + p * (TW / PX)]);
          const float4* w4 = reinterpret_cast<const float4*>(wr + (a * 11 + bb) * COUT);
#pragma unroll
          for (int c4 = 0; c4 < CO_T / 4; ++c4) {
            const float4 w = w4[c4];
            const uint64_t w01 = f32x2_pack(w.x, w.y), w23 = f32x2_pack(w.z, w.w);
#pragma unroll
            for (int p = 0; p < PX; ++p) {
              ffma2(part[p][2 * c4], xv[p], w01);
              ffma2(part[p][2 * c4 + 1], xv[p], w23);
            }
          }
        }
      }
#pragma unroll
      for (int p = 0; p < PX; ++p)
#pragma unroll
        for (int c = 0; c < CO_T / 2; ++c) {
          float lo, hi;
          f32x2_unpack(part[p][c], lo, hi);
          acc[p][2 * c] += lo, acc[p][2 * c + 1] += hi;
        }
    }
  }
  // epilogue: bias, ReLU, store NHWC (CO_T contiguous channels per pixel)
#pragma unroll
  for (int p = 0; p < PX; ++p) {
    const int oy = y0 + py, ox = x0 + pxb + p * (TW / PX);
    if (oy >= n1 || ox >= n2) continue;
    const size_t pix = ((size_t)b * n1 + oy) * n2 + ox;
    float v[CO_T];
#pragma unroll
    for (int c = 0; c < CO_T; ++c) {
      const int co = cg * CO_T + c;
      float bv = 0.f;
      if (bias) bv = fullmap ? bias[((size_t)oy * n2 + ox) * COUT + co] : bias[co];
      v[c] = acc[p][c] + bv;
      if (relu) v[c] = fmaxf(v[c], 0.f);
      if (mask && !(static_cast<float>(mask[pix * COUT + co]) > 0.f)) v[c] = 0.f;   // backward: ReLU'(forward)
    }
    Tout* dst = out + pix * COUT + cg * CO_T;
    if constexpr (sizeof(Tout) == 2) {
#pragma unroll
      for (int c8 = 0; c8 < CO_T / 8; ++c8) {
        uint4 u;
        __nv_bfloat162 h0 = __floats2bfloat162_rn(v[8 * c8 + 0], v[8 * c8 + 1]);
        __nv_bfloat162 h1 = __floats2bfloat162_rn(v[8 * c8 + 2], v[8 * c8 + 3]);
        __nv_bfloat162 h2 = __floats2bfloat162_rn(v[8 * c8 + 4], v[8 * c8 + 5]);
        __nv_bfloat162 h3 = __floats2bfloat162_rn(v[8 * c8 + 6], v[8 * c8 + 7]);
        u.x = *reinterpret_cast<uint32_t*>(&h0), u.y = *reinterpret_cast<uint32_t*>(&h1);
        u.z = *reinterpret_cast<uint32_t*>(&h2), u.w = *reinterpret_cast<uint32_t*>(&h3);
        reinterpret_cast<uint4*>(dst)[c8] = u;
      }
    } else {
#pragma unroll
      for (int c4 = 0; c4 < CO_T / 4; ++c4)
        reinterpret_cast<float4*>(dst)[c4] = make_float4(v[4 * c4], v[4 * c4 + 1], v[4 * c4 + 2], v[4 * c4 + 3]);
    }
  }
}

template <typename Tin, typename Tout, int CIN, int COUT, int CO_T, int CI_CHUNK>
static cudaError_t launch_wide(const void* in, const float* wx, const float* bias, int fullmap, int relu, void* out,
                               int batch, int n1, int n2, cudaStream_t st, const void* mask = nullptr) {
  constexpr int TH = 8, TW = 32;
  const size_t smem = (size_t)(CI_CHUNK * (TH + 10) * 72 + CI_CHUNK * 121 * COUT) * sizeof(float);   // WTS = 72
  auto k = k_conv_wide<Tin, Tout, CIN, COUT, CO_T, CI_CHUNK>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((n2 + TW - 1) / TW, (n1 + TH - 1) / TH, batch);
  k<<<grid, 256, smem, st>>>(reinterpret_cast<const Tin*>(in), wx, bias, fullmap, reinterpret_cast<const Tout*>(mask),
                             relu, reinterpret_cast<Tout*>(out), n1, n2);
  return cudaGetLastError();
}

cudaError_t launch_conv1_simt(const void* xt, bool bf16, const float* wx, const float* bias, int fullmap, void* h1,
                              int batch, int n1, int n2, cudaStream_t st) {
  if (bf16)
    return launch_wide<__nv_bfloat16, __nv_bfloat16, 1, 64, 16, 1>(xt, wx, bias, fullmap, 1, h1, batch, n1, n2, st);
  return launch_wide<float, float, 1, 64, 16, 1>(xt, wx, bias, fullmap, 1, h1, batch, n1, n2, st);
}

// training (k_train.cu): 'same' cross-correlations that transport gradients back through conv layers 3 and 2,
// masked by ReLU'(forward activation): d_out[p][co] = 1(mask > 0) * sum wt[ci][a][b][co] d_in[p + (a-5, b-5)][ci]
cudaError_t launch_dgrad3_f32(const float* dxhat, const float* wt3, const float* h2, float* dh2, int batch, int n1,
                              int n2, cudaStream_t st) {
  return launch_wide<float, float, 1, 32, 8, 1>(dxhat, wt3, nullptr, 0, 0, dh2, batch, n1, n2, st, h2);
}
cudaError_t launch_dgrad2_f32(const float* dh2, const float* wt2, const float* h1, float* dh1, int batch, int n1,
                              int n2, cudaStream_t st) {
  return launch_wide<float, float, 32, 64, 16, 2>(dh2, wt2, nullptr, 0, 0, dh1, batch, n1, n2, st, h1);
}

// custom stacks: the same kernel for the other supported widths, bias + ReLU
cudaError_t launch_convg_simt(int cin, int cout, const float* in, const float* wx, const float* bias, float* out,
                              int batch, int n1, int n2, cudaStream_t st) {
  if (cin == 1 && cout == 32) return launch_wide<float, float, 1, 32, 8, 1>(in, wx, bias, 0, 1, out, batch, n1, n2, st);
  if (cin == 1 && cout == 64) return launch_wide<float, float, 1, 64, 16, 1>(in, wx, bias, 0, 1, out, batch, n1, n2, st);
  if (cin == 32 && cout == 32) return launch_wide<float, float, 32, 32, 8, 2>(in, wx, bias, 0, 1, out, batch, n1, n2, st);
  if (cin == 32 && cout == 64) return launch_wide<float, float, 32, 64, 16, 2>(in, wx, bias, 0, 1, out, batch, n1, n2, st);
  if (cin == 64 && cout == 32) return launch_wide<float, float, 64, 32, 8, 2>(in, wx, bias, 0, 1, out, batch, n1, n2, st);
  if (cin == 64 && cout == 64) return launch_wide<float, float, 64, 64, 16, 2>(in, wx, bias, 0, 1, out, batch, n1, n2, st);
  // width 128 (custom stacks, NEXT-3)
  if (cin == 32 && cout == 128) return launch_wide<float, float, 32, 128, 32, 1>(in, wx, bias, 0, 1, out, batch, n1, n2, st);
  if (cin == 64 && cout == 128) return launch_wide<float, float, 64, 128, 32, 1>(in, wx, bias, 0, 1, out, batch, n1, n2, st);
  if (cin == 128 && cout == 128) return launch_wide<float, float, 128, 128, 32, 1>(in, wx, bias, 0, 1, out, batch, n1, n2, st);
  if (cin == 128 && cout == 64) return launch_wide<float, float, 128, 64, 16, 2>(in, wx, bias, 0, 1, out, batch, n1, n2, st);
  if (cin == 128 && cout == 32) return launch_wide<float, float, 128, 32, 8, 2>(in, wx, bias, 0, 1, out, batch, n1, n2, st);
  return cudaErrorInvalidValue;
}

// custom stacks (NEXT-3), the data gradient of layer (cin -> cout): dX = [X > 0] * correlation of dG (cout channels)
// with the rotated, transposed bank wt [cout][a][b][cin] -- a cout -> cin 'same' layer with a ReLU' mask, no bias
cudaError_t launch_dgrad_simt(int cin, int cout, const float* dG, const float* wt, const float* X, float* dX, int batch,
                              int n1, int n2, cudaStream_t st) {
  if (cout == 32 && cin == 32) return launch_wide<float, float, 32, 32, 8, 2>(dG, wt, nullptr, 0, 0, dX, batch, n1, n2, st, X);
  if (cout == 32 && cin == 64) return launch_wide<float, float, 32, 64, 16, 2>(dG, wt, nullptr, 0, 0, dX, batch, n1, n2, st, X);
  if (cout == 64 && cin == 32) return launch_wide<float, float, 64, 32, 8, 2>(dG, wt, nullptr, 0, 0, dX, batch, n1, n2, st, X);
  if (cout == 64 && cin == 64) return launch_wide<float, float, 64, 64, 16, 2>(dG, wt, nullptr, 0, 0, dX, batch, n1, n2, st, X);
  if (cout == 128 && cin == 32) return launch_wide<float, float, 128, 32, 8, 2>(dG, wt, nullptr, 0, 0, dX, batch, n1, n2, st, X);
  if (cout == 128 && cin == 64) return launch_wide<float, float, 128, 64, 16, 2>(dG, wt, nullptr, 0, 0, dX, batch, n1, n2, st, X);
  if (cout == 128 && cin == 128) return launch_wide<float, float, 128, 128, 32, 1>(dG, wt, nullptr, 0, 0, dX, batch, n1, n2, st, X);
  if (cout == 64 && cin == 128) return launch_wide<float, float, 64, 128, 32, 1>(dG, wt, nullptr, 0, 0, dX, batch, n1, n2, st, X);
  if (cout == 32 && cin == 128) return launch_wide<float, float, 32, 128, 32, 1>(dG, wt, nullptr, 0, 0, dX, batch, n1, n2, st, X);
  if (cout == 1 && cin == 32) return launch_wide<float, float, 1, 32, 8, 1>(dG, wt, nullptr, 0, 0, dX, batch, n1, n2, st, X);
  return cudaErrorInvalidValue;
}

cudaError_t launch_conv2_simt_f32(const float* h1, const float* wx, const float* bias, int fullmap, float* h2,
                                  int batch, int n1, int n2, cudaStream_t st) {
  return launch_wide<float, float, 64, 32, 8, 4>(h1, wx, bias, fullmap, 1, h2, batch, n1, n2, st);
}

// ---------------------------------------------------------------------------------------------
// conv layer 3 (32 -> 1): one output pixel per thread, block 8 x 32 pixels; the halo tile keeps all 32
// input channels per pixel (bf16 inputs stay bf16 in smem, 80-B pixel stride -> conflict-free 16-B reads).
template <typename Tin>
__global__ void __launch_bounds__(256)
    k_conv3(const Tin* __restrict__ in, const float* __restrict__ wx, const float* __restrict__ bias, int fullmap,
            int relu, float* __restrict__ out, int n1, int n2) {
  constexpr int TH = 8, TW = 32, HT = TH + 10, WT = TW + 10, CIN = 32;
  constexpr int PSTR = (sizeof(Tin) == 2) ? 40 : 36;   // padded channel stride (elements)
  extern __shared__ __align__(16) uint8_t sm3[];
  Tin* sx = reinterpret_cast<Tin*>(sm3);                // [HT][WT][PSTR]
  float* sw = reinterpret_cast<float*>(sm3 + (size_t)HT * WT * PSTR * sizeof(Tin));   // [121][32]
  const int b = blockIdx.z, y0 = blockIdx.y * TH, x0 = blockIdx.x * TW;
  const int tid = threadIdx.x;
  constexpr int VEC = 16 / sizeof(Tin);                 // elements per 16-B vector
  for (int e = tid; e < HT * WT * (CIN / VEC); e += 256) {
    const int pix = e / (CIN / VEC), v = e - pix * (CIN / VEC);
    const int yy = pix / WT, xx = pix - yy * WT;
    const int gy = y0 + yy - 5, gx = x0 + xx - 5;
    uint4 val = make_uint4(0, 0, 0, 0);
    if (gy >= 0 && gy < n1 && gx >= 0 && gx < n2)
      val = *reinterpret_cast<const uint4*>(in + (((size_t)b * n1 + gy) * n2 + gx) * CIN + v * VEC);
    *reinterpret_cast<uint4*>(sx + (size_t)pix * PSTR + v * VEC) = val;
  }
  for (int e = tid; e < 121 * CIN; e += 256) {
    const int tap = e / CIN, ci = e - tap * CIN;
    sw[e] = wx[(size_t)ci * 121 + tap];    // wx[ci][tap][co=0] -> sw[tap][ci]
  }
  __syncthreads();
  const int py = tid / TW, px = tid % TW;
  float acc = 0.f;
  for (int c8 = 0; c8 < CIN / 8; ++c8) {
    float part = 0.f;
#pragma unroll 1
    for (int a = 0; a < 11; ++a) {
#pragma unroll
      for (int bb = 0; bb < 11; ++bb) {
        const Tin* xp = sx + ((size_t)(py + a) * WT + px + bb) * PSTR + c8 * 8;
        const float4* wp = reinterpret_cast<const float4*>(sw + (a * 11 + bb) * CIN + c8 * 8);
        const float4 w0 = wp[0], w1 = wp[1];
        float xv[8];
        if constexpr (sizeof(Tin) == 2) {
          const uint4 u = *reinterpret_cast<const uint4*>(xp);
          const uint32_t uw[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            xv[2 * i] = __uint_as_float(uw[i] << 16);
            xv[2 * i + 1] = __uint_as_float(uw[i] & 0xFFFF0000u);
          }
        } else {
          const float4 u0 = reinterpret_cast<const float4*>(xp)[0], u1 = reinterpret_cast<const float4*>(xp)[1];
          xv[0] = u0.x, xv[1] = u0.y, xv[2] = u0.z, xv[3] = u0.w, xv[4] = u1.x, xv[5] = u1.y, xv[6] = u1.z, xv[7] = u1.w;
        }
        part = fmaf(xv[0], w0.x, part);
        part = fmaf(xv[1], w0.y, part);
        part = fmaf(xv[2], w0.z, part);
        part = fmaf(xv[3], w0.w, part);
        part = fmaf(xv[4], w1.x, part);
        part = fmaf(xv[5], w1.y, part);
        part = fmaf(xv[6], w1.z, part);
        part = fmaf(xv[7], w1.w, part);
      }
    }
    acc += part;
  }
  const int oy = y0 + py, ox = x0 + px;
  if (oy < n1 && ox < n2) {
    float bv = 0.f;
    if (bias) bv = fullmap ? bias[(size_t)oy * n2 + ox] : bias[0];
    float v = acc + bv;
    if (relu) v = fmaxf(v, 0.f);
    out[((size_t)b * n1 + oy) * n2 + ox] = v;
  }
}

// fp32 conv layer 3 (32 -> 1), register-blocked sliding window: block = 32 output rows x 64 columns, thread = 8
// consecutive columns of one row.  Channels pass in chunks of 4 through a [4][42][76] halo tile; per (channel, tap
// row) the thread's 18 inputs arrive by 4 LDS.128 + 1 LDS.64 and feed 8 x 11 FMAs (the one-pixel-per-thread
// kernel above re-reads every input from shared memory for each tap and is bound by it).  Accumulation: per channel
// over its 121 taps, then over the 32 channels in order.
constexpr int C3F_TH = 32, C3F_TW = 64, C3F_CC = 4, C3F_WS = 76;
__global__ void __launch_bounds__(256) k_conv3_f32_sw(const float* __restrict__ in, const float* __restrict__ wx,
                                                      const float* __restrict__ bias, int fullmap, int relu,
                                                      float* __restrict__ out, int n1, int n2) {
  constexpr int HT = C3F_TH + 10, WT = C3F_TW + 10;
  extern __shared__ __align__(16) float smf[];
  float* sx = smf;                                   // [C3F_CC][HT][C3F_WS]
  float* sw = smf + C3F_CC * HT * C3F_WS;            // [32 ci][11 a][12] (tap 11 zero)
  const int b = blockIdx.z, y0 = blockIdx.y * C3F_TH, x0 = blockIdx.x * C3F_TW;
  const int tid = threadIdx.x, tx = tid & 7, ty = tid >> 3;
  for (int e = tid; e < 32 * 11 * 12; e += 256) {
    const int ci = e / 132, r = e - ci * 132, a = r / 12, bb = r - a * 12;
    sw[e] = bb < 11 ? wx[(size_t)ci * 121 + a * 11 + bb] : 0.f;
  }
  float acc[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) acc[p] = 0.f;
  for (int cc0 = 0; cc0 < 32; cc0 += C3F_CC) {
    __syncthreads();
    for (int e = tid; e < C3F_CC * HT * WT; e += 256) {   // channel innermost: one pixel's 4 channels per 4 threads
      const int c = e % C3F_CC, pix = e / C3F_CC, yy = pix / WT, xx = pix - yy * WT;
      const int gy = y0 + yy - 5, gx = x0 + xx - 5;
      sx[(c * HT + yy) * C3F_WS + xx] =
          (gy >= 0 && gy < n1 && gx >= 0 && gx < n2) ? in[(((size_t)b * n1 + gy) * n2 + gx) * 32 + cc0 + c] : 0.f;
    }
    __syncthreads();
#pragma unroll 1
    for (int c = 0; c < C3F_CC; ++c) {
      float part[8];
#pragma unroll
      for (int p = 0; p < 8; ++p) part[p] = 0.f;
#pragma unroll 1
      for (int a = 0; a < 11; ++a) {
        const float* xr = sx + (c * HT + ty + a) * C3F_WS + 8 * tx;
        float xv[18];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 v = reinterpret_cast<const float4*>(xr)[q];
          xv[4 * q] = v.x, xv[4 * q + 1] = v.y, xv[4 * q + 2] = v.z, xv[4 * q + 3] = v.w;
        }
        {
          const float2 v = reinterpret_cast<const float2*>(xr)[8];
          xv[16] = v.x, xv[17] = v.y;
        }
        const float4* w4 = reinterpret_cast<const float4*>(sw + ((cc0 + c) * 11 + a) * 12);
        const float4 wa = w4[0], wb = w4[1], wc = w4[2];
        const float w[11] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w, wc.x, wc.y, wc.z};
#pragma unroll
        for (int bb = 0; bb < 11; ++bb)
#pragma unroll
          for (int p = 0; p < 8; ++p) part[p] = fmaf(xv[p + bb], w[bb], part[p]);
      }
#pragma unroll
      for (int p = 0; p < 8; ++p) acc[p] += part[p];
    }
  }
  const int oy = y0 + ty;
  if (oy >= n1) return;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int ox = x0 + 8 * tx + p;
    if (ox >= n2) continue;
    float bv = 0.f;
    if (bias) bv = fullmap ? bias[(size_t)oy * n2 + ox] : bias[0];
    float v = acc[p] + bv;
    if (relu) v = fmaxf(v, 0.f);
    out[((size_t)b * n1 + oy) * n2 + ox] = v;
  }
}

cudaError_t launch_conv3_simt(const void* h2, bool bf16, const float* wx, const float* bias, int fullmap, int relu,
                              float* xhat, int batch, int n1, int n2, cudaStream_t st) {
  if (!bf16) {
    const size_t smem = ((size_t)C3F_CC * (C3F_TH + 10) * C3F_WS + 32 * 11 * 12) * sizeof(float);
    cudaError_t e = cudaFuncSetAttribute(k_conv3_f32_sw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((n2 + C3F_TW - 1) / C3F_TW, (n1 + C3F_TH - 1) / C3F_TH, batch);
    k_conv3_f32_sw<<<grid, 256, smem, st>>>(reinterpret_cast<const float*>(h2), wx, bias, fullmap, relu, xhat, n1, n2);
    return cudaGetLastError();
  }
  constexpr int TH = 8, TW = 32;
  dim3 grid((n2 + TW - 1) / TW, (n1 + TH - 1) / TH, batch);
  if (bf16) {
    const size_t smem = (size_t)(TH + 10) * (TW + 10) * 40 * 2 + 121 * 32 * 4;
    cudaError_t e = cudaFuncSetAttribute(k_conv3<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_conv3<__nv_bfloat16><<<grid, 256, smem, st>>>(reinterpret_cast<const __nv_bfloat16*>(h2), wx, bias, fullmap,
                                                    relu, xhat, n1, n2);
  } else {
    const size_t smem = (size_t)(TH + 10) * (TW + 10) * 36 * 4 + 121 * 32 * 4;
    cudaError_t e = cudaFuncSetAttribute(k_conv3<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_conv3<float><<<grid, 256, smem, st>>>(reinterpret_cast<const float*>(h2), wx, bias, fullmap, relu, xhat, n1,
                                            n2);
  }
  return cudaGetLastError();
}

}  // namespace di
