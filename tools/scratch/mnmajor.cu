// standalone probe: tcgen05.mma kind::tf32 with BOTH operands MN-major (SWIZZLE_128B), MN atoms at arbitrary
// strides (A: row-tap stride PA rows; B: overlapping atoms one 128-B row apart) and K windows starting at
// arbitrary rows.  The layout the TC weight-gradient kernel relies on.
//   strip S: rows of 32 fp32 (128 B), SW128 by address.  A[g*32+i][k] = S[a0 + g*PA + k][i] (4 atoms, M = 128),
//   B[k][t*32+j] = S2[b0 + t + k][j] (NA atoms, N = 32*NA), D = sum over KS K-steps of 8 rows.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include "../../paper_1701_03891_b200/csrc/sm100.cuh"
using namespace di;

constexpr int ROWS = 256;

__global__ void k(const float* S, const float* S2, int a0, int PA, int b0, int NA, int KS, int swap, float* D, int raw) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;
  uint8_t* sB = sm + ROWS * 128;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int e = threadIdx.x; e < ROWS * 32; e += blockDim.x) {
    const int r = e / 32, c = e % 32;
    const int off = r * 128 + (((c / 4) ^ (r & 7)) << 4) + (c % 4) * 4;
    *reinterpret_cast<float*>(sA + (raw ? e * 4 : off)) = S[e];
    *reinterpret_cast<float*>(sB + (raw ? e * 4 : off)) = S2[e];
  }
  fence_async_smem();
  if (threadIdx.x == 0) mbar_init(&bar, 1), fence_mbar_init();
  if (threadIdx.x < 32) tmem_alloc<256>(&tslot), tmem_relinquish();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int N = 32 * NA;
  if (threadIdx.x == 0) {
    const uint32_t id = swap == 2 ? idesc_f32acc(2, 128, N, 0, 0) : idesc_f32acc(2, 128, N, 1, 1);
    if (swap == 2) {   // control: K-major both, A rows m at 128 B, B rows n at 128 B, K = first 8 floats
      umma_tf32_ss(tmem, smem_desc(smem_u32(sA), 16, 1024, kSwizzle128B), smem_desc(smem_u32(sB), 16, 1024, kSwizzle128B),
                   id, 0);
      KS = 0;
    }
    for (int ks = 0; ks < KS; ++ks) {
      const uint32_t la = PA * 128, lb = 128;
      const uint64_t ad = swap ? smem_desc(smem_u32(sA + (a0 + 8 * ks) * 128), 1024, la, kSwizzle128B)
                               : smem_desc(smem_u32(sA + (a0 + 8 * ks) * 128), la, 1024, kSwizzle128B);
      const uint64_t bd = swap ? smem_desc(smem_u32(sB + (b0 + 8 * ks) * 128), 1024, lb, kSwizzle128B)
                               : smem_desc(smem_u32(sB + (b0 + 8 * ks) * 128), lb, 1024, kSwizzle128B);
      umma_tf32_ss(tmem, ad, bd, id, ks > 0);
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  for (int c = 0; c < N; c += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + ((uint32_t)(w * 32) << 16) + c, r);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) D[(w * 32 + l) * 256 + c + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<256>(tmem);
}

#include <cuda_bf16.h>
__global__ void kb(const float* S, const float* S2, int a0, int PA, int b0, int NA, int KS, int swap, float* D) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;
  uint8_t* sB = sm + ROWS * 128;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int e = threadIdx.x; e < ROWS * 64; e += blockDim.x) {
    const int r = e / 64, c = e % 64;
    const int off = r * 128 + (((c / 8) ^ (r & 7)) << 4) + (c % 8) * 2;
    *reinterpret_cast<__nv_bfloat16*>(sA + off) = __float2bfloat16(S[e]);
    *reinterpret_cast<__nv_bfloat16*>(sB + off) = __float2bfloat16(S2[e]);
  }
  fence_async_smem();
  if (threadIdx.x == 0) mbar_init(&bar, 1), fence_mbar_init();
  if (threadIdx.x < 32) tmem_alloc<256>(&tslot), tmem_relinquish();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int N = 64 * NA;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_f32acc(1, 128, N, 1, 1);
    for (int ks = 0; ks < KS; ++ks) {
      const uint32_t la = PA * 128, lb = 128;
      const uint64_t ad = swap ? smem_desc(smem_u32(sA + (a0 + 16 * ks) * 128), 1024, la, kSwizzle128B)
                               : smem_desc(smem_u32(sA + (a0 + 16 * ks) * 128), la, 1024, kSwizzle128B);
      const uint64_t bd = swap ? smem_desc(smem_u32(sB + (b0 + 16 * ks) * 128), 1024, lb, kSwizzle128B)
                               : smem_desc(smem_u32(sB + (b0 + 16 * ks) * 128), lb, 1024, kSwizzle128B);
      umma_f16_ss(tmem, ad, bd, id, ks > 0);
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  for (int c = 0; c < N; c += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + ((uint32_t)(w * 32) << 16) + c, r);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) D[(w * 32 + l) * 256 + c + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<256>(tmem);
}
__global__ void kb2(const float* S, const float* S2, int a0, int PA, int b0, int NA, int KS, float* D) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;
  uint8_t* sB = sm + ROWS * 128;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int e = threadIdx.x; e < ROWS * 64; e += blockDim.x) {
    const int r = e / 64, c = e % 64;
    *reinterpret_cast<__nv_bfloat16*>(sA + r * 128 + (((c / 8) ^ (r & 7)) << 4) + (c % 8) * 2) = __float2bfloat16(S[e]);
  }
  for (int e = threadIdx.x; e < ROWS * 32; e += blockDim.x) {   // SW64: 16-B chunk ^= (addr >> 7) & 3
    const int r = e / 32, c = e % 32;
    const int lin = r * 64 + (c / 8) * 16;
    const int phys = lin ^ (((lin >> 7) & 3) << 4);
    *reinterpret_cast<__nv_bfloat16*>(sB + phys + (c % 8) * 2) = __float2bfloat16(S2[e]);
  }
  fence_async_smem();
  if (threadIdx.x == 0) mbar_init(&bar, 1), fence_mbar_init();
  if (threadIdx.x < 32) tmem_alloc<256>(&tslot), tmem_relinquish();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int N = 32 * NA;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_f32acc(1, 128, N, 1, 1);
    for (int ks = 0; ks < KS; ++ks) {
      const uint64_t ad = smem_desc(smem_u32(sA + (a0 + 16 * ks) * 128), PA * 128, 1024, kSwizzle128B);
      const uint64_t bd = smem_desc(smem_u32(sB + (b0 + 16 * ks) * 64), 64, 512, kSwizzle64B);
      umma_f16_ss(tmem, ad, bd, id, ks > 0);
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  for (int c = 0; c < N; c += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + ((uint32_t)(w * 32) << 16) + c, r);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) D[(w * 32 + l) * 256 + c + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<256>(tmem);
}
// generic MN-major probe: A rows of RA bytes (SWA swizzle), M = 128 as NA_M atoms of RA/2 elements at stride PA
// rows; B rows of RB bytes, N = RB/2 (one atom).  A[g*EA + i][k] = SA[a0 + g*PA + k][i], B[k][j] = SB[b0 + k][j]
__device__ __forceinline__ uint32_t swz(uint32_t lin, int R) {   // address-based swizzle of byte offset lin
  if (R == 128) return lin ^ (((lin >> 7) & 7) << 4);
  if (R == 64) return lin ^ (((lin >> 7) & 3) << 4);
  return lin ^ (((lin >> 7) & 1) << 4);
}
__global__ void kg(const float* S, const float* S2, int RA, int RB, int a0, int PA, int b0, int KS, float* D) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;
  uint8_t* sB = sm + ROWS * 128;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int EA = RA / 2, EB = RB / 2;
  for (int e = threadIdx.x; e < ROWS * EA; e += blockDim.x) {
    const int r = e / EA, c = e % EA;
    const uint32_t lin = r * RA + (c / 8) * 16;
    *reinterpret_cast<__nv_bfloat16*>(sA + swz(lin, RA) + (c % 8) * 2) = __float2bfloat16(S[e]);
  }
  for (int e = threadIdx.x; e < ROWS * EB; e += blockDim.x) {
    const int r = e / EB, c = e % EB;
    const uint32_t lin = r * RB + (c / 8) * 16;
    *reinterpret_cast<__nv_bfloat16*>(sB + swz(lin, RB) + (c % 8) * 2) = __float2bfloat16(S2[e]);
  }
  fence_async_smem();
  if (threadIdx.x == 0) mbar_init(&bar, 1), fence_mbar_init();
  if (threadIdx.x < 32) tmem_alloc<256>(&tslot), tmem_relinquish();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t lay = [](int R) { return R == 128 ? kSwizzle128B : R == 64 ? kSwizzle64B : kSwizzle32B; }(RA);
  const uint32_t layb = RB == 128 ? kSwizzle128B : RB == 64 ? kSwizzle64B : kSwizzle32B;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_f32acc(1, 128, EB, 1, 1);
    for (int ks = 0; ks < KS; ++ks) {
      const uint64_t ad = smem_desc(smem_u32(sA + (a0 + 16 * ks) * RA), PA * RA, 8 * RA, lay);
      const uint64_t bd = smem_desc(smem_u32(sB + (b0 + 16 * ks) * RB), RB, 8 * RB, layb);
      umma_f16_ss(tmem, ad, bd, id, ks > 0);
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  for (int c = 0; c < EB; c += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + ((uint32_t)(w * 32) << 16) + c, r);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) D[(w * 32 + l) * 256 + c + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<256>(tmem);
}
static float bfr(float x) { return __bfloat162float(__float2bfloat16(x)); }

static float tf(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u &= ~0x1FFFu;
  float y;
  memcpy(&y, &u, 4);
  return y;
}

int main() {
  std::vector<float> S(ROWS * 32), S2(ROWS * 32);
  uint64_t st = 12345;
  auto rnd = [&]() {
    st = st * 6364136223846793005ULL + 1442695040888963407ULL;
    return (float)((st >> 40) & 0xFFFF) / 65536.f - 0.5f;
  };
  for (auto& v : S) v = rnd();
  std::vector<float> S0 = S;
  for (auto& v : S2) v = rnd();
  float *dS, *dS2, *dD;
  cudaMalloc(&dS, S.size() * 4), cudaMalloc(&dS2, S2.size() * 4), cudaMalloc(&dD, 128 * 256 * 4);
  cudaMemcpy(dS, S.data(), S.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dS2, S2.data(), S2.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * ROWS * 128 + 1024);
  {  // diagnostic: A raw slot i holds value i (i < 2048), B one-hot at raw slot sb
    std::vector<float> A(ROWS * 32, 0.f), B(ROWS * 32, 0.f);
    for (int i = 0; i < 2048; ++i) A[i] = (float)i;
    cudaMemcpy(dS, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 2; ++mode)
    for (int sb : {0, 1, 4, 32, 64, 96, 128, 224, 256, 1024}) {
      std::fill(B.begin(), B.end(), 0.f);
      B[sb] = 1.f;
      cudaMemcpy(dS2, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
      cudaMemset(dD, 0, 128 * 256 * 4);
      k<<<1, 128, 2 * ROWS * 128 + 1024>>>(dS, dS2, 0, 8, 0, 8, 1, mode, dD, 1);
      cudaDeviceSynchronize();
      std::vector<float> D(128 * 256);
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      printf("mode %d B raw slot %d -> cols:", mode, sb);
      int shown = 0;
      for (int n = 0; n < 256; ++n) {
        bool nz = false;
        for (int m = 0; m < 128; ++m) nz |= D[m * 256 + n] != 0.f;
        if (nz && shown < 6) {
          printf(" n=%d[A m0..3: %g %g %g %g m8:%g m31:%g m32:%g m64:%g]", n, D[0 * 256 + n], D[1 * 256 + n], D[2 * 256 + n],
                 D[3 * 256 + n], D[8 * 256 + n], D[31 * 256 + n], D[32 * 256 + n], D[64 * 256 + n]);
          ++shown;
        }
        if (nz && shown >= 6) ++shown;
      }
      printf(" (total %d)\n", shown);
    }
  }
  struct C { int a0, PA, b0, NA, KS; } cases[] = {{0, 8, 0, 8, 1}, {3, 13, 5, 8, 1}, {3, 13, 5, 8, 4}, {7, 37, 1, 3, 3},
                                                  {1, 21, 2, 6, 5}};
  cudaMemcpy(dS, S.data(), S.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dS2, S2.data(), S2.size() * 4, cudaMemcpyHostToDevice);
  {
    cudaMemset(dD, 0, 128 * 256 * 4);
    k<<<1, 128, 2 * ROWS * 128 + 1024>>>(dS, dS2, 0, 8, 0, 8, 1, 2, dD, 0);
    printf("control: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    std::vector<float> D(128 * 256);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, mx = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 256; ++n) {
        double ref = 0;
        for (int kk = 0; kk < 8; ++kk) ref += (double)tf(S[m * 32 + kk]) * tf(S2[n * 32 + kk]);
        maxerr = fmax(maxerr, fabs(ref - D[m * 256 + n])), mx = fmax(mx, fabs(D[m * 256 + n]));
      }
    printf("control K-major maxerr=%.3g max|D|=%.3g\n", maxerr, mx);
  }
  for (int swap = 0; swap < 2; ++swap)
    for (auto cs : cases) {
      cudaMemset(dD, 0, 128 * 256 * 4);
      k<<<1, 128, 2 * ROWS * 128 + 1024>>>(dS, dS2, cs.a0, cs.PA, cs.b0, cs.NA, cs.KS, swap, dD, 0);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("swap=%d case a0=%d: %s\n", swap, cs.a0, cudaGetErrorString(e));
        return 1;
      }
      std::vector<float> D(128 * 256);
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      double maxerr = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 32 * cs.NA; ++n) {
          const int g = m / 32, i = m % 32, t = n / 32, j = n % 32;
          double ref = 0;
          for (int kk = 0; kk < 8 * cs.KS; ++kk)
            ref += (double)tf(S[(cs.a0 + g * cs.PA + kk) * 32 + i]) * tf(S2[(cs.b0 + t + kk) * 32 + j]);
          maxerr = fmax(maxerr, fabs(ref - D[m * 256 + n]));
        }
      double mx = 0;
      for (float v : D) mx = fmax(mx, fabs(v));
      printf("max|D|=%.3g ", mx);
      printf("swap=%d a0=%d PA=%d b0=%d NA=%d KS=%d maxerr=%.3g %s\n", swap, cs.a0, cs.PA, cs.b0, cs.NA, cs.KS, maxerr,
             maxerr < 1e-3 ? "OK" : "BAD");
    }
  cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * ROWS * 128 + 1024);
  {
    std::vector<float> A(ROWS * 64), B(ROWS * 64);
    for (auto& v : A) v = rnd();
    for (auto& v : B) v = rnd();
    float *dA, *dB;
    cudaMalloc(&dA, A.size() * 4), cudaMalloc(&dB, B.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    struct C { int a0, PA, b0, NA, KS; } cb[] = {{0, 16, 0, 1, 1}, {0, 16, 0, 4, 1}, {3, 21, 5, 4, 2}};
    for (int swap = 0; swap < 2; ++swap)
      for (auto cs : cb) {
        cudaMemset(dD, 0, 128 * 256 * 4);
        kb<<<1, 128, 2 * ROWS * 128 + 1024>>>(dA, dB, cs.a0, cs.PA, cs.b0, cs.NA, cs.KS, swap, dD);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> D(128 * 256);
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double maxerr = 0, mx = 0;
        for (int m = 0; m < 128; ++m)
          for (int n = 0; n < 64 * cs.NA; ++n) {
            const int g = m / 64, i = m % 64, t = n / 64, j = n % 64;
            double ref = 0;
            for (int kk = 0; kk < 16 * cs.KS; ++kk)
              ref += (double)bfr(A[(cs.a0 + g * cs.PA + kk) * 64 + i]) * bfr(B[(cs.b0 + t + kk) * 64 + j]);
            maxerr = fmax(maxerr, fabs(ref - D[m * 256 + n])), mx = fmax(mx, fabs(D[m * 256 + n]));
          }
        printf("bf16 %s swap=%d a0=%d PA=%d b0=%d NA=%d KS=%d maxerr=%.3g max|D|=%.3g\n", cudaGetErrorString(e), swap,
               cs.a0, cs.PA, cs.b0, cs.NA, cs.KS, maxerr, mx);
      }
  }
  cudaFuncSetAttribute(kb2, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * ROWS * 128 + 1024);
  {
    std::vector<float> A(ROWS * 64), B(ROWS * 32);
    for (auto& v : A) v = rnd();
    for (auto& v : B) v = rnd();
    float *dA, *dB;
    cudaMalloc(&dA, A.size() * 4), cudaMalloc(&dB, B.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    struct C { int a0, PA, b0, NA, KS; } cb[] = {{0, 16, 0, 1, 1}, {0, 16, 0, 8, 1}, {3, 21, 5, 8, 2}, {2, 74, 9, 3, 3},
                                                 {10, 74, 1, 8, 5}};
    for (auto cs : cb) {
      cudaMemset(dD, 0, 128 * 256 * 4);
      kb2<<<1, 128, 2 * ROWS * 128 + 1024>>>(dA, dB, cs.a0, cs.PA, cs.b0, cs.NA, cs.KS, dD);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<float> D(128 * 256);
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      double maxerr = 0, mx = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 32 * cs.NA; ++n) {
          const int g = m / 64, i = m % 64, t = n / 32, j = n % 32;
          double ref = 0;
          for (int kk = 0; kk < 16 * cs.KS; ++kk)
            ref += (double)bfr(A[(cs.a0 + g * cs.PA + kk) * 64 + i]) * bfr(B[(cs.b0 + t + kk) * 32 + j]);
          maxerr = fmax(maxerr, fabs(ref - D[m * 256 + n])), mx = fmax(mx, fabs(D[m * 256 + n]));
        }
      printf("kb2 %s a0=%d PA=%d b0=%d NA=%d KS=%d maxerr=%.3g max|D|=%.3g\n", cudaGetErrorString(e), cs.a0, cs.PA,
             cs.b0, cs.NA, cs.KS, maxerr, mx);
    }
  }
  cudaFuncSetAttribute(kg, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * ROWS * 128 + 1024);
  {
    std::vector<float> A(ROWS * 64), B(ROWS * 64);
    for (auto& v : A) v = rnd();
    for (auto& v : B) v = rnd();
    float *dA, *dB;
    cudaMalloc(&dA, A.size() * 4), cudaMalloc(&dB, B.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    struct C { int RA, RB, a0, PA, b0, KS; } cb[] = {{32, 128, 0, 16, 0, 1}, {32, 128, 3, 21, 5, 3}, {32, 128, 1, 74, 9, 4},
                                                     {64, 32, 0, 16, 0, 1}, {64, 32, 3, 21, 5, 3}, {64, 32, 2, 40, 7, 4},
                                                     {128, 32, 5, 33, 2, 3}};
    for (auto cs : cb) {
      cudaMemset(dD, 0, 128 * 256 * 4);
      kg<<<1, 128, 2 * ROWS * 128 + 1024>>>(dA, dB, cs.RA, cs.RB, cs.a0, cs.PA, cs.b0, cs.KS, dD);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<float> D(128 * 256);
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      const int EA = cs.RA / 2, EB = cs.RB / 2;
      double maxerr = 0, mx = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < EB; ++n) {
          const int g = m / EA, i = m % EA;
          double ref = 0;
          for (int kk = 0; kk < 16 * cs.KS; ++kk)
            ref += (double)bfr(A[(cs.a0 + g * cs.PA + kk) * EA + i]) * bfr(B[(cs.b0 + kk) * EB + n]);
          maxerr = fmax(maxerr, fabs(ref - D[m * 256 + n])), mx = fmax(mx, fabs(D[m * 256 + n]));
        }
      printf("kg %s RA=%d RB=%d a0=%d PA=%d b0=%d KS=%d maxerr=%.3g max|D|=%.3g\n", cudaGetErrorString(e), cs.RA, cs.RB,
             cs.a0, cs.PA, cs.b0, cs.KS, maxerr, mx);
    }
  }
  return 0;
}
