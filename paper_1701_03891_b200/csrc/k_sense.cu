// k_sense.cu -- the sensing model and the quality metrics around the recovery path:
//   measurement      y = Phi x                                   (§1)
//   noise            y + w, w ~ N(0, sigma^2 I) per image, 10 log10(||y||^2 / E||w||^2) = snr_db
//                    (Table 3; measurement-domain reading, DESIGN.md §2 Q14)
//   metrics          PSNR = 10 log10(max(x)^2 / MSE), NMSE = ||x_hat - x||^2 / ||x||^2 and the
//                    success indicator NMSE <= 0.1, per image, accumulated in fp64.
// The sensing GEMM itself reuses the tcgen05 GEMM of k_proxy.cu (roles of the operands swapped); this file holds
// the element-wise / per-image kernels and the fp32 SIMT sensing GEMM.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace di {

// ----------------------------------------------------------------------------- staging for the sensing GEMM
// x [B][N] fp32 -> [B][ldo] in the storage type, zero in columns N..ldo-1 (the K-major A operand of the sensing GEMM)
template <typename T>
__global__ void k_stage_x(const float* __restrict__ x, int N, int ldo, long long count, T* __restrict__ out) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < count; e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / ldo;
    const int j = (int)(e - b * ldo);
    const float v = j < N ? x[b * N + j] : 0.f;
    if constexpr (sizeof(T) == 2)
      out[e] = __float2bfloat16_rn(v);
    else
      out[e] = v;
  }
}

cudaError_t launch_stage_x(const float* x, int N, int ldo, int batch, void* out, bool bf16, cudaStream_t st) {
  const long long count = (long long)batch * ldo, blocks = (count + 255) / 256;
  const int g = (int)(blocks < 8192 ? blocks : 8192);
  if (bf16)
    k_stage_x<__nv_bfloat16><<<g, 256, 0, st>>>(x, N, ldo, count, reinterpret_cast<__nv_bfloat16*>(out));
  else
    k_stage_x<float><<<g, 256, 0, st>>>(x, N, ldo, count, reinterpret_cast<float*>(out));
  return cudaGetLastError();
}

// Phi^T [N][kpad] (storage type) -> Phi [m][ldp] (storage type, zero columns N..ldp-1): the row-major copy the
// sensing GEMM reads K-major
template <typename T>
__global__ void k_untranspose(const T* __restrict__ phiT, int m, int N, int kpad, int tr, int ldp, T* __restrict__ phi) {
  __shared__ T tile[32][33];
  const int j0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int j = j0 + r, i = i0 + threadIdx.x;
    tile[r][threadIdx.x] = (j < N && i < m) ? phiT[phiT_blk_index(j, i, kpad, 128 / (int)sizeof(T), tr)] : T(0);
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int i = i0 + r, j = j0 + threadIdx.x;
    if (i < m && j < ldp) phi[(size_t)i * ldp + j] = j < N ? tile[threadIdx.x][r] : T(0);
  }
}

cudaError_t launch_untranspose(const void* phiT, int m, int N, int kpad, int tr, int ldp, void* phi, bool bf16,
                               cudaStream_t st) {
  dim3 grid((ldp + 31) / 32, (m + 31) / 32), block(32, 8);
  if (bf16)
    k_untranspose<uint16_t><<<grid, block, 0, st>>>(reinterpret_cast<const uint16_t*>(phiT), m, N, kpad, tr, ldp,
                                                    reinterpret_cast<uint16_t*>(phi));
  else
    k_untranspose<float><<<grid, block, 0, st>>>(reinterpret_cast<const float*>(phiT), m, N, kpad, tr, ldp,
                                                 reinterpret_cast<float*>(phi));
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- fp32 sensing GEMM (SIMT)
// y[b][i] = sum_j x[b][j] * phi[i][j]: 64 (b) x 64 (i) tile, 256 threads, 4x4 outputs each, two-level
// accumulation (per 16-wide K chunk, then total) for the fp32 path's 1e-5 bar.
__global__ void __launch_bounds__(256) k_measure_f32(const float* __restrict__ x, const float* __restrict__ phi,
                                                     int m, int N, int batch, float* __restrict__ y, long long ldy) {
  __shared__ float sx[16][64 + 4];
  __shared__ float sp[16][64 + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int i0 = blockIdx.x * 64, b0 = blockIdx.y * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < N; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int r = e / 16, kk = e % 16;     // coalesced along K
      const int k = k0 + kk;
      sx[kk][r] = (b0 + r < batch && k < N) ? x[(size_t)(b0 + r) * N + k] : 0.f;
      sp[kk][r] = (i0 + r < m && k < N) ? phi[(size_t)(i0 + r) * N + k] : 0.f;
    }
    __syncthreads();
    float part[4][4] = {};
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], bv[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) a[t] = sx[kk][ty * 4 + t], bv[t] = sp[kk][tx + 16 * t];
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int q = 0; q < 4; ++q) part[t][q] = fmaf(a[t], bv[q], part[t][q]);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[t][q] += part[t][q];
    __syncthreads();
  }
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int b = b0 + ty * 4 + t;
    if (b >= batch) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + tx + 16 * q;
      if (i < m) y[(size_t)b * ldy + i] = acc[t][q];
    }
  }
}

cudaError_t launch_measure_f32(const float* x, const float* phi, int m, int N, int batch, float* y, long long ldy,
                               cudaStream_t st) {
  dim3 grid((m + 63) / 64, (batch + 63) / 64);
  k_measure_f32<<<grid, 256, 0, st>>>(x, phi, m, N, batch, y, ldy);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- measurement noise
// splitmix64 (Steele, Lea, Flood 2014) on key + (counter + 1) * golden, 53-bit uniforms, Box-Muller (cosine
// branch): the counter-based generator of synth/rng.py, re-implemented here so that standard normal i of the
// stream is the same number on both sides.
__device__ __forceinline__ uint64_t sm64_mix(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}
__device__ __forceinline__ double sm64_uniform(uint64_t key, uint64_t i) {
  return (double)(sm64_mix(key + (i + 1) * 0x9E3779B97F4A7C15ull) >> 11) * (1.0 / 9007199254740992.0);
}
__device__ __forceinline__ double sm64_normal(uint64_t key, uint64_t i) {
  const double u1 = 1.0 - sm64_uniform(key, 2 * i), u2 = sm64_uniform(key, 2 * i + 1);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

template <typename T>
__device__ __forceinline__ double ld_d(const T* p);
template <>
__device__ __forceinline__ double ld_d<float>(const float* p) { return (double)*p; }
template <>
__device__ __forceinline__ double ld_d<__nv_bfloat16>(const __nv_bfloat16* p) { return (double)__bfloat162float(*p); }

__device__ __forceinline__ void st_t(float* p, double v) { *p = (float)v; }
__device__ __forceinline__ void st_t(__nv_bfloat16* p, double v) { *p = __float2bfloat16_rn((float)v); }

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
  return t;
}

// one block per image: sigma^2 = ||y_b||^2 / (m * 10^(snr/10)); y_b[i] += sigma * z(b*m + i)
template <typename T>
__global__ void __launch_bounds__(256) k_add_noise(T* __restrict__ y, long long ldy, int m, double snr_lin,
                                                   uint64_t key) {
  __shared__ double red[8];
  T* yb = y + (size_t)blockIdx.x * ldy;
  double e = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double v = ld_d(yb + i);
    e += v * v;
  }
  e = block_sum(e, red);
  const double sigma = sqrt(e / ((double)m * snr_lin));
  for (int i = threadIdx.x; i < m; i += blockDim.x)
    st_t(yb + i, ld_d(yb + i) + sigma * sm64_normal(key, (uint64_t)blockIdx.x * m + i));
}

cudaError_t launch_add_noise(void* y, long long ldy, int m, int batch, double snr_db, uint64_t key, bool bf16,
                             cudaStream_t st) {
  const double snr_lin = pow(10.0, snr_db / 10.0);
  if (bf16)
    k_add_noise<__nv_bfloat16><<<batch, 256, 0, st>>>(reinterpret_cast<__nv_bfloat16*>(y), ldy, m, snr_lin, key);
  else
    k_add_noise<float><<<batch, 256, 0, st>>>(reinterpret_cast<float*>(y), ldy, m, snr_lin, key);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- metrics
// one block per image; out[b] = PSNR (dB, +inf when MSE = 0), out[B + b] = NMSE, out[2B + b] = success (0/1)
__global__ void __launch_bounds__(256) k_metrics(const float* __restrict__ xhat, const float* __restrict__ x, int N,
                                                 int batch, double* __restrict__ out) {
  __shared__ double red[8];
  __shared__ float redm[8];
  const float* xh = xhat + (size_t)blockIdx.x * N;
  const float* xb = x + (size_t)blockIdx.x * N;
  double se = 0.0, sx = 0.0;
  float mx = -INFINITY;
  const bool vec = (N % 4) == 0;   // rows 16-B aligned: float4 loads (HBM-bound pass)
  const int n4 = vec ? N / 4 : 0;
  for (int j = threadIdx.x; j < n4; j += blockDim.x) {
    const float4 h = __ldg(reinterpret_cast<const float4*>(xh) + j), t = __ldg(reinterpret_cast<const float4*>(xb) + j);
    const double d0 = (double)h.x - t.x, d1 = (double)h.y - t.y, d2 = (double)h.z - t.z, d3 = (double)h.w - t.w;
    se += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
    sx += (double)t.x * t.x + (double)t.y * t.y + (double)t.z * t.z + (double)t.w * t.w;
    mx = fmaxf(mx, fmaxf(fmaxf(t.x, t.y), fmaxf(t.z, t.w)));
  }
  for (int j = 4 * n4 + threadIdx.x; j < N; j += blockDim.x) {
    const double d = (double)xh[j] - (double)xb[j];
    se += d * d;
    sx += (double)xb[j] * (double)xb[j];
    mx = fmaxf(mx, xb[j]);
  }
  se = block_sum(se, red);
  sx = block_sum(sx, red);
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) redm[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = redm[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) m = fmaxf(m, redm[i]);
    const double mse = se / N, peak = (double)m;
    out[blockIdx.x] = mse == 0.0 ? INFINITY : 10.0 * log10(peak * peak / mse);
    const double nmse = se / sx;
    out[batch + blockIdx.x] = nmse;
    out[2 * batch + blockIdx.x] = nmse <= 0.1 ? 1.0 : 0.0;
  }
}

cudaError_t launch_metrics(const float* xhat, const float* x, int N, int batch, double* out, cudaStream_t st) {
  k_metrics<<<batch, 256, 0, st>>>(xhat, x, N, batch, out);
  return cudaGetLastError();
}

}  // namespace di
