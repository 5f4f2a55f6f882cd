// tools/ladder.cu -- hardware probe for the sm_100a features the DeepInverse kernels rely on.
// Not part of the product.  Build: make -C tools ladder ; run on a B200: tools/ladder [test...]
//
//   t1  TMEM alloc + tcgen05.st/ld round trip (address = lane<<16 | column)
//   t2  SS UMMA M=128, N in {16..256}, K=64, SWIZZLE_128B K-major operands vs host
//   t3  A-operand window starting at an arbitrary 128-B row (base_offset field)
//   t4  TS UMMA: A in TMEM
//   t5  TMA 4-D box with negative coordinates (OOB zero fill) + SWIZZLE_128B layout
//   t6  UMMA throughput (SS / TS, N sweep, with and without TMA ingest)
//   t7  .ws MMA exploration (M=32/64/128): D layout, collector reuse, B shift
//   t8  collector::a reuse throughput
//   t16 disable-output-lane masks of tcgen05.mma (per-lane keep / overwrite / accumulate)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../paper_1701_03891_b200/csrc/sm100.cuh"

using namespace di;

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) {                                                            \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

__device__ int g_err;

__device__ __forceinline__ void wait_bounded(uint64_t* bar, uint32_t parity) {
  long long n = 0;
  while (!mbar_try_wait(bar, parity)) {
    if (++n > (1ll << 26)) {
      atomicExch(&g_err, 1);
      return;
    }
  }
}

// write a [rows][64] bf16 row-major matrix into smem in the SWIZZLE_128B K-major layout
// (chunk c of row r stored at r*128 + ((c ^ (r & 7)) << 4); base must be 1024-aligned)
__device__ void st_sw128(uint8_t* base, const __nv_bfloat16* g, int rows) {
  for (int idx = threadIdx.x; idx < rows * 8; idx += blockDim.x) {
    int r = idx >> 3, c = idx & 7;
    uint4 v = reinterpret_cast<const uint4*>(g)[r * 8 + c];
    *reinterpret_cast<uint4*>(base + r * 128 + ((c ^ (r & 7)) << 4)) = v;
  }
}

// dump TMEM lanes 0..127, columns [0, ncols) to global (fp32 bits), 4 warps
__device__ void dump_tmem(uint32_t tbase, float* out, int ncols) {
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (w >= 4) return;
  for (int c = 0; c < ncols; c += 16) {
    uint32_t r[16];
    tmem_ld16(tbase + ((uint32_t)(w * 32) << 16) + c, r);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) out[(size_t)(w * 32 + l) * ncols + c + j] = __uint_as_float(r[j]);
  }
}

// ------------------------------------------------------------------------ t1
__global__ void k_t1(float* out) {
  __shared__ uint32_t tslot;
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (w == 0) tmem_alloc<512>(&tslot), tmem_relinquish();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tb = tslot;
  for (int c = 0; c < 512; c += 16) {
    uint32_t r[16];
    for (int j = 0; j < 16; ++j) r[j] = __float_as_uint((float)((w * 32 + l) * 1000 + c + j));
    tmem_st16(tb + ((uint32_t)(w * 32) << 16) + c, r);
  }
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  dump_tmem(tb, out, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (w == 0) tmem_dealloc<512>(tb);
}

// ------------------------------------------------------------------------ t2/t3/t4
// A: [arows][64] bf16 (arows <= 256), B: [N][64]; D = A[a0 : a0+128] * B^T.
// mode 0: SS with base_offset = bo_mode ? (start>>7)&7 : 0 ; mode 1: TS (A staged in TMEM via tcgen05.st)
__global__ void k_mma1(const __nv_bfloat16* A, int arows, const __nv_bfloat16* B, int N, int a0, int bo_mode,
                       int mode, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;               // 32 KB
  uint8_t* sB = smem + 32768;       // 32 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  int w = threadIdx.x >> 5;
  st_sw128(sA, A, arows);
  st_sw128(sB, B, N);
  fence_async_smem();
  if (w == 0) tmem_alloc<512>(&tslot), tmem_relinquish();
  if (threadIdx.x == 32) mbar_init(&bar, 1), fence_mbar_init();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tb = tslot;
  const uint32_t acc_col = 256;  // D at columns 256..; A (TS) at columns 0..31
  if (mode == 1 && w < 4) {
    // TS: A row r -> lane r, K pairs packed into 32-bit columns (k even in the low half)
    int r = w * 32 + (threadIdx.x & 31) + a0;
    uint32_t v[16];
    for (int half = 0; half < 2; ++half) {
      for (int j = 0; j < 16; ++j) {
        int k = (half * 16 + j) * 2;
        __nv_bfloat16 lo = A[r * 64 + k], hi = A[r * 64 + k + 1];
        v[j] = (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
      }
      tmem_st16(tb + ((uint32_t)(w * 32) << 16) + half * 16, v);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    uint32_t idesc = idesc_f32acc(1, 128, N);
    for (int k = 0; k < 4; ++k) {
      uint32_t sa = smem_u32(sA) + a0 * 128 + k * 32;
      uint32_t sb = smem_u32(sB) + k * 32;
      uint64_t ad = smem_desc(sa, 16, 1024, kSwizzle128B, bo_mode ? ((sa >> 7) & 7) : 0);
      uint64_t bd = smem_desc(sb, 16, 1024, kSwizzle128B, 0);
      if (mode == 0)
        umma_f16_ss(tb + acc_col, ad, bd, idesc, k > 0);
      else
        umma_f16_ts(tb + acc_col, tb + k * 8, bd, idesc, k > 0);
    }
    umma_commit(&bar);
  }
  wait_bounded(&bar, 0);
  tc_fence_after();
  dump_tmem(tb + acc_col, out, N);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (w == 0) tmem_dealloc<512>(tb);
}

// ------------------------------------------------------------------------ t5
__global__ void k_t5(const __grid_constant__ CUtensorMap map, int c1, int c2, int c3, uint8_t* out, int bytes) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, bytes);
    tma_load_4d(smem, &map, &bar, 0, c1, c2, c3);
  }
  wait_bounded(&bar, 0);
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) out[i] = smem[i];
}

// ------------------------------------------------------------------------ t6 throughput
// Every CTA: one thread issues `iters` x 4 MMAs (K=64 per group) into one accumulator.
// mode 0 SS, 1 TS, 2 SS with collector::a fill/use/lastuse over pairs of D (A reuse).
// ingest: warps 4..7 stream `ingest` bytes per chunk with cp.async.bulk from an L2-resident buffer.
__global__ void __launch_bounds__(256, 1)
    k_thr(int N, int mode, int iters, const uint8_t* src, int ingest, unsigned long long* cyc, unsigned long long* bytes_in) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;              // 16 KB (128 x 64 bf16)
  uint8_t* sB = smem + 16384;      // 32 KB (256 x 64)
  uint8_t* sI = smem + 49152;      // ingest landing zone (up to 96 KB)
  __shared__ uint64_t bar, ibar;
  __shared__ uint32_t tslot;
  __shared__ volatile int done;
  int w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 49152 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  fence_async_smem();
  if (w == 0) tmem_alloc<512>(&tslot), tmem_relinquish();
  if (threadIdx.x == 32) mbar_init(&bar, 1), mbar_init(&ibar, 1), fence_mbar_init();
  if (threadIdx.x == 0) done = 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    uint32_t idesc = idesc_f32acc(1, 128, N);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int k = 0; k < 4; ++k) {
        uint64_t ad = smem_desc(smem_u32(sA) + k * 32, 16, 1024, kSwizzle128B);
        uint64_t bd = smem_desc(smem_u32(sB) + k * 32, 16, 1024, kSwizzle128B);
        if (mode == 0) {
          umma_f16_ss(tb, ad, bd, idesc, 1);
        } else if (mode == 1) {
          umma_f16_ts(tb + 256, tb + k * 8, bd, idesc, 1);
        } else {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16.collector::a::fill [%0], %1, %2, %3, p;\n\t}" ::"r"(tb),
              "l"(ad), "l"(bd), "r"(idesc), "r"(1));
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16.collector::a::lastuse [%0], %1, %2, %3, p;\n\t}" ::"r"(tb + 256),
              "l"(ad), "l"(bd), "r"(idesc), "r"(1));
        }
      }
    }
    umma_commit(&bar);
    wait_bounded(&bar, 0);
    unsigned long long t1 = clock64();
    done = 1;
    cyc[blockIdx.x] = t1 - t0;
  } else if (w >= 4 && ingest > 0) {
    if (threadIdx.x == 128) {
      unsigned long long got = 0;
      uint32_t ph = 0;
      const uint8_t* s = src + (size_t)(blockIdx.x % 16) * 1048576;
      while (!done) {
        mbar_arrive_expect_tx(&ibar, ingest);
        for (int off = 0; off < ingest; off += 16384) bulk_load(sI + off, s + off, 16384, &ibar);
        wait_bounded(&ibar, ph);
        ph ^= 1;
        got += ingest;
      }
      bytes_in[blockIdx.x] = got;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (w == 0) tmem_dealloc<512>(tb);
}

// ------------------------------------------------------------------------ t7 .ws
// D = A[M x 16] * B[N x 16]^T with .ws (collector b0).  A rows in SW128 tile (K=64 stored, first 16 used).
// variant 0: fill only; 1: fill with B1 then 'use' with descriptor of B2 (collector reuse probe);
// 2: mask descriptor with shift s (nzm=1 -> mask disabled) ; 3: throughput loop
__global__ void k_ws(const __nv_bfloat16* A, const __nv_bfloat16* B1, const __nv_bfloat16* B2, int M, int N,
                     int variant, uint64_t mask_desc, int iters, float* out, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB1 = smem + 32768;
  uint8_t* sB2 = smem + 65536;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  int w = threadIdx.x >> 5;
  st_sw128(sA, A, 128);
  st_sw128(sB1, B1, 256);
  st_sw128(sB2, B2, 256);
  fence_async_smem();
  if (w == 0) tmem_alloc<512>(&tslot), tmem_relinquish();
  if (threadIdx.x == 32) mbar_init(&bar, 1), fence_mbar_init();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tb = tslot;
  // pre-fill TMEM with -1 so untouched cells are visible
  if (w < 4) {
    uint32_t r[16];
    for (int j = 0; j < 16; ++j) r[j] = __float_as_uint(-1.0f);
    for (int c = 0; c < 512; c += 16) tmem_st16(tb + ((uint32_t)(w * 32) << 16) + c, r);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    uint32_t idesc = idesc_f32acc(1, M, N) | (variant == 2 ? (2u << 30) : 0u);
    uint64_t ad = smem_desc(smem_u32(sA), 16, 1024, kSwizzle128B);
    uint64_t bd1 = smem_desc(smem_u32(sB1), 16, 1024, kSwizzle128B);
    uint64_t bd2 = smem_desc(smem_u32(sB2), 16, 1024, kSwizzle128B);
    unsigned long long t0 = clock64();
    if (variant == 0) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.ws.cta_group::1.kind::f16.collector::b0::fill [%0], %1, %2, %3, p;\n\t}" ::"r"(tb),
          "l"(ad), "l"(bd1), "r"(idesc), "r"(0));
    } else if (variant == 1) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.ws.cta_group::1.kind::f16.collector::b0::fill [%0], %1, %2, %3, p;\n\t}" ::"r"(tb),
          "l"(ad), "l"(bd1), "r"(idesc), "r"(0));
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.ws.cta_group::1.kind::f16.collector::b0::use [%0], %1, %2, %3, p;\n\t}" ::"r"(tb + 256),
          "l"(ad), "l"(bd2), "r"(idesc), "r"(0));
    } else if (variant == 2) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.ws.cta_group::1.kind::f16.collector::b0::fill [%0], %1, %2, %3, p, %5;\n\t}" ::"r"(tb),
          "l"(ad), "l"(bd1), "r"(idesc), "r"(0), "l"(mask_desc));
    } else {
      for (int it = 0; it < iters; ++it) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.ws.cta_group::1.kind::f16.collector::b0::fill [%0], %1, %2, %3, p;\n\t}" ::"r"(tb),
            "l"(ad), "l"(bd1), "r"(idesc), "r"(1));
        for (int j = 0; j < 3; ++j)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.ws.cta_group::1.kind::f16.collector::b0::use [%0], %1, %2, %3, p;\n\t}" ::"r"(tb),
              "l"(ad), "l"(bd1), "r"(idesc), "r"(1));
      }
    }
    umma_commit(&bar);
    wait_bounded(&bar, 0);
    if (cyc) cyc[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  tc_fence_after();
  if (out && blockIdx.x == 0) dump_tmem(tb, out, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (w == 0) tmem_dealloc<512>(tb);
}

// ============================================================================ host
static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }
static std::vector<__nv_bfloat16> randbf(int n, unsigned seed, std::vector<float>& f) {
  std::vector<__nv_bfloat16> v(n);
  f.resize(n);
  srand(seed);
  for (int i = 0; i < n; ++i) {
    float x = (float)(rand() % 2001 - 1000) / 1000.0f;
    v[i] = __float2bfloat16(x);
    f[i] = __bfloat162float(v[i]);
  }
  return v;
}
template <class T>
static T* dup(const std::vector<T>& h) {
  T* d;
  CK(cudaMalloc(&d, h.size() * sizeof(T)));
  CK(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}
static int check_err(const char* t) {
  int e = 0;
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpyFromSymbol(&e, g_err, sizeof(int)));
  if (e) printf("{\"test\":\"%s\",\"error\":\"mbarrier timeout\"}\n", t);
  int z = 0;
  CK(cudaMemcpyToSymbol(g_err, &z, sizeof(int)));
  return e;
}

static void t1() {
  float* d;
  CK(cudaMalloc(&d, 128 * 512 * 4));
  k_t1<<<1, 128>>>(d);
  check_err("t1");
  std::vector<float> h(128 * 512);
  CK(cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int l = 0; l < 128; ++l)
    for (int c = 0; c < 512; ++c) bad += h[l * 512 + c] != (float)(l * 1000 + c);
  printf("{\"test\":\"t1_tmem_roundtrip\",\"pass\":%s,\"bad\":%d}\n", bad ? "false" : "true", bad);
  cudaFree(d);
}

static double ref_check(const std::vector<float>& Af, const std::vector<float>& Bf, int a0, int N,
                        const std::vector<float>& D) {
  double maxerr = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < 64; ++k) s += (double)Af[(a0 + m) * 64 + k] * Bf[n * 64 + k];
      maxerr = fmax(maxerr, fabs(s - D[m * N + n]));
    }
  return maxerr;
}

static void t234() {
  std::vector<float> Af, Bf;
  auto A = randbf(256 * 64, 1, Af);
  auto B = randbf(256 * 64, 2, Bf);
  __nv_bfloat16 *dA = dup(A), *dB = dup(B);
  float* dD;
  CK(cudaMalloc(&dD, 128 * 256 * 4));
  CK(cudaFuncSetAttribute(k_mma1, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  std::vector<float> D(128 * 256);
  for (int N : {16, 32, 64, 128, 256}) {
    k_mma1<<<1, 128, 65536>>>(dA, 256, dB, N, 0, 0, 0, dD);
    if (check_err("t2")) return;
    CK(cudaMemcpy(D.data(), dD, 128 * N * 4, cudaMemcpyDeviceToHost));
    double e = ref_check(Af, Bf, 0, N, D);
    printf("{\"test\":\"t2_ss_mma\",\"N\":%d,\"maxerr\":%.3g,\"pass\":%s}\n", N, e, e < 1e-3 ? "true" : "false");
  }
  for (int a0 : {0, 1, 3, 5, 8, 13, 74, 127}) {
    for (int bo = 0; bo < 2; ++bo) {
      k_mma1<<<1, 128, 65536>>>(dA, 256, dB, 64, a0, bo, 0, dD);
      if (check_err("t3")) return;
      CK(cudaMemcpy(D.data(), dD, 128 * 64 * 4, cudaMemcpyDeviceToHost));
      double e = ref_check(Af, Bf, a0, 64, D);
      printf("{\"test\":\"t3_shifted_A\",\"a0\":%d,\"base_offset_mode\":%d,\"maxerr\":%.3g,\"pass\":%s}\n", a0, bo,
             e, e < 1e-3 ? "true" : "false");
    }
  }
  for (int N : {32, 64, 256}) {
    k_mma1<<<1, 128, 65536>>>(dA, 256, dB, N, 0, 0, 1, dD);
    if (check_err("t4")) return;
    CK(cudaMemcpy(D.data(), dD, 128 * N * 4, cudaMemcpyDeviceToHost));
    double e = ref_check(Af, Bf, 0, N, D);
    printf("{\"test\":\"t4_ts_mma\",\"N\":%d,\"maxerr\":%.3g,\"pass\":%s}\n", N, e, e < 1e-3 ? "true" : "false");
  }
  cudaFree(dA), cudaFree(dB), cudaFree(dD);
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiled get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  return (EncodeTiled)fn;
}

static void t5() {
  const int Bn = 2, H = 8, W = 8, C = 64;
  std::vector<float> f;
  auto X = randbf(Bn * H * W * C, 5, f);
  __nv_bfloat16* dX = dup(X);
  CUtensorMap map;
  cuuint64_t dims[4] = {C, W, H, Bn};
  cuuint64_t strides[3] = {C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
  cuuint32_t box[4] = {64, 12, 4, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = get_encode()(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, dX, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("{\"test\":\"t5_tma\",\"encode_error\":%d}\n", (int)r);
    return;
  }
  int bytes = 64 * 12 * 4 * 2;
  uint8_t* dout;
  CK(cudaMalloc(&dout, bytes));
  CK(cudaFuncSetAttribute(k_t5, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
  int x0 = -2, y0 = -1, b0 = 1;
  k_t5<<<1, 128, 16384>>>(map, x0, y0, b0, dout, bytes);
  if (check_err("t5")) return;
  std::vector<uint8_t> h(bytes);
  CK(cudaMemcpy(h.data(), dout, bytes, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int yy = 0; yy < 4; ++yy)
    for (int xx = 0; xx < 12; ++xx) {
      int p = yy * 12 + xx;
      int gy = y0 + yy, gx = x0 + xx;
      for (int c = 0; c < 64; ++c) {
        int chunk = (c * 2) >> 4;
        int off = p * 128 + ((chunk ^ (p & 7)) << 4) + (c * 2 & 15);
        uint16_t got = h[off] | (h[off + 1] << 8);
        uint16_t want = 0;
        if (gy >= 0 && gy < H && gx >= 0 && gx < W) {
          __nv_bfloat16 v = X[(((size_t)b0 * H + gy) * W + gx) * C + c];
          want = *reinterpret_cast<uint16_t*>(&v);
        }
        bad += got != want;
      }
    }
  printf("{\"test\":\"t5_tma_oob_sw128\",\"bad\":%d,\"pass\":%s}\n", bad, bad ? "false" : "true");
  cudaFree(dX), cudaFree(dout);
}

static void t6(int nsm) {
  unsigned long long *dc, *db;
  CK(cudaMalloc(&dc, nsm * 8));
  CK(cudaMalloc(&db, nsm * 8));
  uint8_t* src;
  CK(cudaMalloc(&src, 16 << 20));
  CK(cudaMemset(src, 0, 16 << 20));
  CK(cudaFuncSetAttribute(k_thr, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152 + 98304));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  struct Cfg { int N, mode, ingest; };
  std::vector<Cfg> cfgs;
  for (int mode : {0, 1})
    for (int N : {32, 64, 128, 256}) cfgs.push_back({N, mode, 0});
  for (int N : {64, 128, 256}) cfgs.push_back({N, 2, 0});
  for (int ing : {16384, 32768, 65536})
    for (int N : {128, 256}) cfgs.push_back({N, 0, ing});
  for (int ing : {32768, 65536}) cfgs.push_back({256, 1, ing});
  for (auto c : cfgs) {
    int iters = 4096 * 64 / c.N;
    k_thr<<<nsm, 256, 49152 + 98304>>>(c.N, c.mode, 8, src, 0, dc, db);  // warm
    CK(cudaMemset(db, 0, nsm * 8));
    cudaEventRecord(e0);
    k_thr<<<nsm, 256, 49152 + 98304>>>(c.N, c.mode, iters, src, c.ingest, dc, db);
    cudaEventRecord(e1);
    if (check_err("t6")) return;
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> hc(nsm), hb(nsm);
    CK(cudaMemcpy(hc.data(), dc, nsm * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hb.data(), db, nsm * 8, cudaMemcpyDeviceToHost));
    double cmax = 0, bsum = 0;
    for (int i = 0; i < nsm; ++i) cmax = fmax(cmax, (double)hc[i]), bsum += hb[i];
    int per = (c.mode == 2) ? 8 : 4;
    double mmas = (double)iters * per;
    double flops = 2.0 * 128 * c.N * 16 * mmas * nsm;
    double mhz = cmax / (ms * 1e3);
    printf("{\"test\":\"t6_throughput\",\"mode\":\"%s\",\"N\":%d,\"ingest_chunk\":%d,\"cyc_per_mma\":%.2f,"
           "\"floor_cyc\":%.1f,\"tflops\":%.1f,\"mhz\":%.0f,\"ingest_B_per_clk_per_sm\":%.1f}\n",
           c.mode == 0 ? "SS" : (c.mode == 1 ? "TS" : "SS_collA_pair"), c.N, c.ingest, cmax / mmas,
           128.0 * c.N / 256.0, flops / (ms * 1e-3) / 1e12, mhz, bsum / nsm / cmax);
  }
  cudaFree(dc), cudaFree(db), cudaFree(src);
}

static void t7(int nsm) {
  // A[m][0] = m+1, A[m][1] = 1 ; B[n][0] = 1, B[n][1] = 256*(n+1)  => D[m][n] = (m+1) + 256 (n+1)
  std::vector<__nv_bfloat16> A(128 * 64), B1(256 * 64), B2(256 * 64);
  for (auto& v : A) v = __float2bfloat16(0.f);
  for (auto& v : B1) v = __float2bfloat16(0.f);
  for (auto& v : B2) v = __float2bfloat16(0.f);
  for (int m = 0; m < 128; ++m) A[m * 64] = __float2bfloat16((float)(m + 1)), A[m * 64 + 1] = __float2bfloat16(1.f);
  for (int n = 0; n < 256; ++n) {
    B1[n * 64] = __float2bfloat16(1.f), B1[n * 64 + 1] = __float2bfloat16(256.f * (n + 1));
    B2[n * 64] = __float2bfloat16(1.f), B2[n * 64 + 1] = __float2bfloat16(-256.f * (n + 1));
  }
  __nv_bfloat16 *dA = dup(A), *dB1 = dup(B1), *dB2 = dup(B2);
  float* dD;
  CK(cudaMalloc(&dD, 128 * 512 * 4));
  unsigned long long* dc;
  CK(cudaMalloc(&dc, nsm * 8));
  CK(cudaFuncSetAttribute(k_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304));
  std::vector<float> D(128 * 512);
  auto report = [&](const char* name, int M, int N) {
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    // print a compact map: for each lane, first column holding a value != -1 and its decoded (m, n)
    printf("{\"test\":\"%s\",\"M\":%d,\"N\":%d,\"cells\":[", name, M, N);
    int printed = 0;
    for (int l = 0; l < 128; ++l)
      for (int c = 0; c < 512; ++c) {
        float v = D[l * 512 + c];
        if (v == -1.0f) continue;
        if ((c % 16 == 0 && (l % 8 == 0)) || (l < 2 && c < 4)) {
          double vv = v;
          int n1 = (int)floor(vv / 256.0);
          int m1 = (int)(vv - 256.0 * n1);
          printf("%s[%d,%d,%.0f,%d,%d]", printed++ ? "," : "", l, c, v, m1 - 1, n1 - 1);
        }
      }
    int nz = 0;
    for (float v : D) nz += v != -1.0f;
    printf("],\"written\":%d}\n", nz);
  };
  for (int M : {32, 64, 128})
    for (int N : {64, 128, 256}) {
      k_ws<<<1, 128, 98304>>>(dA, dB1, dB2, M, N, 0, 0ull, 0, dD, nullptr);
      if (check_err("t7")) return;
      char nm[64];
      snprintf(nm, 64, "t7_ws_fill");
      report(nm, M, N);
    }
  k_ws<<<1, 128, 98304>>>(dA, dB1, dB2, 32, 128, 1, 0ull, 0, dD, nullptr);
  if (!check_err("t7u")) report("t7_ws_fill_then_use_B2desc(col256+)", 32, 128);
  for (int s : {1, 3}) {
    // MaskAndShiftB: nzm(bit39)=1 disables the mask; shift in bits [56,62)
    uint64_t md = (1ull << 39) | ((uint64_t)s << 56);
    k_ws<<<1, 128, 98304>>>(dA, dB1, dB2, 32, 128, 2, md, 0, dD, nullptr);
    char nm[64];
    snprintf(nm, 64, "t7_ws_shift%d", s);
    if (!check_err("t7s")) report(nm, 32, 128);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  for (int M : {32, 64, 128})
    for (int N : {64, 128, 256}) {
      int iters = 8192;
      cudaEventRecord(e0);
      k_ws<<<nsm, 128, 98304>>>(dA, dB1, dB2, M, N, 3, 0ull, iters, nullptr, dc);
      cudaEventRecord(e1);
      if (check_err("t7t")) return;
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      std::vector<unsigned long long> hc(nsm);
      CK(cudaMemcpy(hc.data(), dc, nsm * 8, cudaMemcpyDeviceToHost));
      double cmax = 0;
      for (auto v : hc) cmax = fmax(cmax, (double)v);
      double mmas = iters * 4.0;
      printf("{\"test\":\"t7_ws_throughput\",\"M\":%d,\"N\":%d,\"cyc_per_mma\":%.2f,\"useful_tflops\":%.1f}\n", M,
             N, cmax / mmas, 2.0 * M * N * 16 * mmas * nsm / (ms * 1e-3) / 1e12);
    }
  cudaFree(dA), cudaFree(dB1), cudaFree(dB2), cudaFree(dD), cudaFree(dc);
}


// ------------------------------------------------------------------------ t9 .ws pipelining / semantics
template <int BUF>
__device__ __forceinline__ void ws_mma(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc, int op,
                                       uint64_t mask) {
  // op 0 fill, 1 use, 2 lastuse, 3 discard ; mask != 0 -> pass zero-column mask descriptor
#define WS_ASM(BS, OPS)                                                                                   \
  if (mask)                                                                                               \
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"                                        \
                 "tcgen05.mma.ws.cta_group::1.kind::f16.collector::" BS "::" OPS " [%0], %1, %2, %3, p, %5;\n\t}" ::"r"(d), \
                 "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "l"(mask));                                       \
  else                                                                                                    \
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"                                        \
                 "tcgen05.mma.ws.cta_group::1.kind::f16.collector::" BS "::" OPS " [%0], %1, %2, %3, p;\n\t}" ::"r"(d), \
                 "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
#define WS_OPS(BS)                              \
  if (op == 0) { WS_ASM(BS, "fill") }           \
  else if (op == 1) { WS_ASM(BS, "use") }       \
  else if (op == 2) { WS_ASM(BS, "lastuse") }   \
  else { WS_ASM(BS, "discard") }
  if (BUF == 0) { WS_OPS("b0") }
  else if (BUF == 1) { WS_OPS("b1") }
  else if (BUF == 2) { WS_OPS("b2") }
  else { WS_OPS("b3") }
#undef WS_OPS
#undef WS_ASM
}
__device__ __forceinline__ void ws_any(int buf, uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc,
                                       int op, uint64_t mask) {
  switch (buf) {
    case 0: ws_mma<0>(d, ad, bd, idesc, acc, op, mask); break;
    case 1: ws_mma<1>(d, ad, bd, idesc, acc, op, mask); break;
    case 2: ws_mma<2>(d, ad, bd, idesc, acc, op, mask); break;
    default: ws_mma<3>(d, ad, bd, idesc, acc, op, mask); break;
  }
}
// throughput: NACC accumulators (each its own collector buffer), REUSE MMAs per fill, all compile-time
// KIND 0 = ws, 1 = plain SS (M=128), 2 = TS (M=128)
template <int KIND, int M, int N, int NACC, int REUSE, bool MASK>
__global__ void __launch_bounds__(128, 1) k_pipe(int iters, uint64_t mask, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  int w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  fence_async_smem();
  if (w == 0) tmem_alloc<512>(&tslot), tmem_relinquish();
  if (threadIdx.x == 32) mbar_init(&bar, 1), fence_mbar_init();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_f32acc(1, M, N) | (MASK ? (2u << 30) : 0u);
    constexpr uint32_t dcols = (KIND == 0) ? (M == 32 ? N / 4 : (M == 64 ? N / 2 : N)) : N;
    uint64_t ad[REUSE], bd[NACC];
#pragma unroll
    for (int r = 0; r < REUSE; ++r) ad[r] = smem_desc(smem_u32(smem) + (r & 3) * 32, 16, 1024, kSwizzle128B);
#pragma unroll
    for (int a = 0; a < NACC; ++a) bd[a] = smem_desc(smem_u32(smem) + 32768 + (a & 1) * 16384, 16, 1024, kSwizzle128B);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < REUSE; ++r) {
#pragma unroll
        for (int a = 0; a < NACC; ++a) {
          const uint32_t d = tb + a * dcols;
          if constexpr (KIND == 0) {
            constexpr int dummy = 0; (void)dummy;
            const int op = (REUSE == 1) ? 3 : (r == 0 ? 0 : (r == REUSE - 1 ? 2 : 1));
            if (a == 0) ws_mma<0>(d, ad[r], bd[a], idesc, 1, op, MASK ? mask : 0);
            else if (a == 1) ws_mma<1>(d, ad[r], bd[a], idesc, 1, op, MASK ? mask : 0);
            else if (a == 2) ws_mma<2>(d, ad[r], bd[a], idesc, 1, op, MASK ? mask : 0);
            else ws_mma<3>(d, ad[r], bd[a], idesc, 1, op, MASK ? mask : 0);
          } else if constexpr (KIND == 1) {
            umma_f16_ss(d, ad[r], bd[a], idesc, 1);
          } else {
            umma_f16_ts(tb + a * N, tb + 448 + (r & 3) * 8, bd[a], idesc, 1);
          }
        }
      }
    }
    umma_commit(&bar);
    wait_bounded(&bar, 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (w == 0) tmem_dealloc<512>(tb);
}

template <int KIND, int M, int N, int NACC, int REUSE, bool MASK>
static void run_pipe(int nsm, unsigned long long* dc, uint64_t mask) {
  auto k = k_pipe<KIND, M, N, NACC, REUSE, MASK>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  int iters = 16384 / (NACC * REUSE) * 4;
  k<<<nsm, 128, 98304>>>(16, mask, dc);
  cudaEventRecord(e0);
  k<<<nsm, 128, 98304>>>(iters, mask, dc);
  cudaEventRecord(e1);
  if (check_err("t9")) return;
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<unsigned long long> hc(nsm);
  CK(cudaMemcpy(hc.data(), dc, nsm * 8, cudaMemcpyDeviceToHost));
  double cmax = 0;
  for (auto v : hc) cmax = fmax(cmax, (double)v);
  double mmas = (double)iters * NACC * REUSE;
  printf("{\"test\":\"t9_pipe\",\"kind\":\"%s\",\"M\":%d,\"N\":%d,\"nacc\":%d,\"reuse\":%d,\"mask\":%d,"
         "\"cyc_per_mma\":%.2f,\"frac_of_8192\":%.3f,\"tflops\":%.0f,\"mhz\":%.0f}\n",
         KIND == 0 ? "ws" : (KIND == 1 ? "SS" : "TS"), M, N, NACC, REUSE, (int)MASK, cmax / mmas,
         2.0 * M * N * 16 / (cmax / mmas) / 8192.0, 2.0 * M * N * 16 * mmas * nsm / (ms * 1e-3) / 1e12,
         cmax / (ms * 1e3));
}

static void t9(int nsm) {
  unsigned long long* dc;
  CK(cudaMalloc(&dc, nsm * 8));
  uint64_t mk = (1ull << 39) | ((uint64_t)3 << 56) | (59ull << 48) | (3ull << 40);  // mask on, shift 3
  run_pipe<0, 32, 256, 1, 4, false>(nsm, dc, 0);
  run_pipe<0, 32, 256, 2, 4, false>(nsm, dc, 0);
  run_pipe<0, 32, 256, 4, 4, false>(nsm, dc, 0);
  run_pipe<0, 32, 256, 1, 1, false>(nsm, dc, 0);
  run_pipe<0, 32, 256, 4, 1, false>(nsm, dc, 0);
  run_pipe<0, 32, 256, 1, 11, false>(nsm, dc, 0);
  run_pipe<0, 32, 256, 2, 11, false>(nsm, dc, 0);
  run_pipe<0, 32, 256, 4, 11, false>(nsm, dc, 0);
  run_pipe<0, 32, 256, 2, 11, true>(nsm, dc, mk);
  run_pipe<0, 32, 256, 4, 11, true>(nsm, dc, mk);
  run_pipe<0, 32, 128, 4, 11, false>(nsm, dc, 0);
  run_pipe<0, 64, 256, 1, 4, false>(nsm, dc, 0);
  run_pipe<0, 64, 256, 2, 4, false>(nsm, dc, 0);
  run_pipe<0, 64, 256, 2, 11, true>(nsm, dc, mk);
  run_pipe<0, 64, 128, 4, 11, false>(nsm, dc, 0);
  run_pipe<0, 128, 256, 1, 4, false>(nsm, dc, 0);
  run_pipe<0, 128, 256, 2, 4, false>(nsm, dc, 0);
  run_pipe<1, 128, 64, 1, 4, false>(nsm, dc, 0);
  run_pipe<1, 128, 64, 2, 4, false>(nsm, dc, 0);
  run_pipe<1, 128, 64, 4, 4, false>(nsm, dc, 0);
  run_pipe<1, 128, 128, 1, 4, false>(nsm, dc, 0);
  run_pipe<1, 128, 128, 2, 4, false>(nsm, dc, 0);
  run_pipe<1, 128, 256, 1, 4, false>(nsm, dc, 0);
  run_pipe<1, 128, 256, 2, 4, false>(nsm, dc, 0);
  run_pipe<2, 128, 128, 1, 4, false>(nsm, dc, 0);
  run_pipe<2, 128, 128, 2, 4, false>(nsm, dc, 0);
  run_pipe<2, 128, 256, 1, 4, false>(nsm, dc, 0);
  cudaFree(dc);
}

// semantics: B rows n = 0..255 carry value n+1 in k=1 (A[m][1] = 1) ; print full D row m=0 for each quadrant
__global__ void k_sem(const __nv_bfloat16* A, const __nv_bfloat16* B, int M, int N, uint64_t mask, int bufop, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + 32768;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  int w = threadIdx.x >> 5;
  st_sw128(sA, A, 128);
  st_sw128(sB, B, 320);
  fence_async_smem();
  if (w == 0) tmem_alloc<512>(&tslot), tmem_relinquish();
  if (threadIdx.x == 32) mbar_init(&bar, 1), fence_mbar_init();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tb = tslot;
  if (w < 4) {
    uint32_t r[16];
    for (int j = 0; j < 16; ++j) r[j] = __float_as_uint(-1.0f);
    for (int c = 0; c < 512; c += 16) tmem_st16(tb + ((uint32_t)(w * 32) << 16) + c, r);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    uint32_t idesc = idesc_f32acc(1, M, N) | (2u << 30);
    uint64_t ad = smem_desc(smem_u32(sA), 16, 1024, kSwizzle128B);
    uint64_t bd = smem_desc(smem_u32(sB), 16, 1024, kSwizzle128B);
    if (bufop == 0) {
      ws_mma<0>(tb, ad, bd, idesc, 0, 0, mask);
    } else {
      // fill without shift, then 'use' with the mask/shift -> is the shift applied to the collector copy?
      ws_mma<0>(tb + 256, ad, bd, idesc, 0, 0, 0);
      ws_mma<0>(tb, ad, bd, idesc, 0, 2, mask);
    }
    umma_commit(&bar);
    wait_bounded(&bar, 0);
  }
  __syncthreads();
  tc_fence_after();
  dump_tmem(tb, out, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (w == 0) tmem_dealloc<512>(tb);
}

static void t10() {
  std::vector<__nv_bfloat16> A(128 * 64), B(320 * 64);
  for (auto& v : A) v = __float2bfloat16(0.f);
  for (auto& v : B) v = __float2bfloat16(0.f);
  for (int m = 0; m < 128; ++m) A[m * 64 + 1] = __float2bfloat16(1.f);
  for (int n = 0; n < 320; ++n) B[n * 64 + 1] = __float2bfloat16((float)(n + 1));
  __nv_bfloat16 *dA = dup(A), *dB = dup(B);
  float* dD;
  CK(cudaMalloc(&dD, 128 * 512 * 4));
  CK(cudaFuncSetAttribute(k_sem, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304));
  std::vector<float> D(128 * 512);
  struct S { int M, N; uint64_t mask; int bufop; const char* name; };
  auto mk = [](int shift, int nzm, int use, int skip, int first, int s0, int s1, int s2, int s3) {
    return (uint64_t)(s0 & 255) | ((uint64_t)(s1 & 255) << 8) | ((uint64_t)(s2 & 255) << 16) |
           ((uint64_t)(s3 & 255) << 24) | ((uint64_t)(first & 15) << 32) | ((uint64_t)nzm << 39) |
           ((uint64_t)((skip - 1) & 255) << 40) | ((uint64_t)((use - 1) & 255) << 48) | ((uint64_t)shift << 56);
  };
  std::vector<S> ss = {
      {32, 256, mk(0, 0, 1, 1, 0, 0, 0, 0, 0), 0, "shift0_nzm0"},
      {32, 256, mk(5, 0, 1, 1, 0, 0, 0, 0, 0), 0, "shift5_nzm0"},
      {32, 256, mk(10, 0, 1, 1, 0, 0, 0, 0, 0), 0, "shift10_nzm0"},
      {32, 256, mk(3, 1, 60, 4, 0, 0, 0, 0, 0), 0, "shift3_use60_skip4_first0_start0"},
      {32, 256, mk(3, 1, 60, 4, 1, 0, 0, 0, 0), 0, "shift3_use60_skip4_first1_start0"},
      {32, 256, mk(3, 1, 60, 4, 0, 2, 2, 2, 2), 0, "shift3_use60_skip4_first0_start2"},
      {32, 256, mk(3, 1, 60, 4, 0, 2, 0, 0, 0), 0, "shift3_use60_skip4_first0_start2_only_q0"},
      {32, 128, mk(7, 0, 1, 1, 0, 0, 0, 0, 0), 0, "N128_shift7_nzm0"},
      {32, 256, mk(4, 0, 1, 1, 0, 0, 0, 0, 0), 1, "fill_noshift_then_lastuse_shift4"},
      {64, 256, mk(3, 0, 1, 1, 0, 0, 0, 0, 0), 0, "M64_shift3_nzm0"},
      {128, 256, mk(3, 0, 1, 1, 0, 0, 0, 0, 0), 0, "M128_shift3_nzm0"},
  };
  for (auto s : ss) {
    k_sem<<<1, 128, 98304>>>(dA, dB, s.M, s.N, s.mask, s.bufop, dD);
    if (check_err("t10")) return;
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    int cols = s.M == 32 ? s.N / 4 : (s.M == 64 ? s.N / 2 : s.N);
    printf("{\"test\":\"t10_%s\",\"M\":%d,\"N\":%d,\"rows\":{", s.name, s.M, s.N);
    int lanes[4] = {0, 32, 64, 96};
    for (int q = 0; q < 4; ++q) {
      printf("%s\"lane%d\":[", q ? "," : "", lanes[q]);
      for (int c = 0; c < cols; ++c) printf("%s%.0f", c ? "," : "", D[lanes[q] * 512 + c]);
      printf("]");
    }
    printf("}}\n");
  }
  cudaFree(dA), cudaFree(dB), cudaFree(dD);
}


// ------------------------------------------------------------------------ t11 / t12: narrow swizzles
// Rows of RB bytes (RB = 32 -> SWIZZLE_32B, 64 -> SWIZZLE_64B, 128 -> SWIZZLE_128B), K = RB/2 bf16 per row.
// Swizzle is applied on absolute smem address bits: 16-B chunk bits [4, 4+log2(RB/16)) ^= bits [7, ...).
__device__ __forceinline__ uint32_t swz_off(uint32_t off, int RB) {
  const uint32_t mask = (RB == 128) ? 7u : (RB == 64 ? 3u : 1u);
  return off ^ (((off >> 7) & mask) << 4);
}
__device__ void st_swz(uint8_t* base, const __nv_bfloat16* g, int rows, int RB) {
  const int cpr = RB / 16;
  for (int idx = threadIdx.x; idx < rows * cpr; idx += blockDim.x) {
    int r = idx / cpr, c = idx % cpr;
    uint4 v = reinterpret_cast<const uint4*>(g)[idx];
    *reinterpret_cast<uint4*>(base + swz_off(r * RB + c * 16, RB)) = v;
  }
}
__host__ __device__ inline uint32_t layout_of(int RB) { return RB == 128 ? 2u : (RB == 64 ? 4u : 6u); }

// D[128][N] = A[a0 : a0+128][K] * B[N][K]^T, A and B in the RB-swizzled layout
__global__ void k_mma_swz(const __nv_bfloat16* A, int arows, const __nv_bfloat16* B, int N, int a0, int RB,
                          float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;             // up to 256 rows x 128 B = 32 KB
  uint8_t* sB = smem + 32768;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  int w = threadIdx.x >> 5;
  st_swz(sA, A, arows, RB);
  st_swz(sB, B, N, RB);
  fence_async_smem();
  if (w == 0) tmem_alloc<512>(&tslot), tmem_relinquish();
  if (threadIdx.x == 32) mbar_init(&bar, 1), fence_mbar_init();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    uint32_t idesc = idesc_f32acc(1, 128, N);
    const int nk = RB / 32;
    const uint32_t sbo = 8 * RB;
    for (int k = 0; k < nk; ++k) {
      uint32_t sa = smem_u32(sA) + a0 * RB + k * 32;
      uint32_t sb = smem_u32(sB) + k * 32;
      umma_f16_ss(tb, smem_desc(sa, 16, sbo, layout_of(RB)), smem_desc(sb, 16, sbo, layout_of(RB)), idesc, k > 0);
    }
    umma_commit(&bar);
  }
  wait_bounded(&bar, 0);
  tc_fence_after();
  dump_tmem(tb, out, N);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (w == 0) tmem_dealloc<512>(tb);
}

static void t11() {
  for (int RB : {32, 64}) {
    const int K = RB / 2;
    std::vector<float> Af, Bf;
    auto A = randbf(256 * K, 11 + RB, Af);
    auto B = randbf(256 * K, 12 + RB, Bf);
    __nv_bfloat16 *dA = dup(A), *dB = dup(B);
    float* dD;
    CK(cudaMalloc(&dD, 128 * 256 * 4));
    CK(cudaFuncSetAttribute(k_mma_swz, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024));
    std::vector<float> D(128 * 256);
    for (int N : {16, 32, 64, 256})
      for (int a0 : {0, 1, 3, 5, 7, 8, 13, 74, 111}) {
        if (a0 + 128 > 256) continue;
        k_mma_swz<<<1, 128, 65536 + 1024>>>(dA, 256, dB, N, a0, RB, dD);
        if (check_err("t11")) return;
        CK(cudaMemcpy(D.data(), dD, 128 * N * 4, cudaMemcpyDeviceToHost));
        double e = 0;
        for (int m = 0; m < 128; ++m)
          for (int n = 0; n < N; ++n) {
            double s = 0;
            for (int k = 0; k < K; ++k) s += (double)Af[(a0 + m) * K + k] * Bf[n * K + k];
            e = fmax(e, fabs(s - D[m * N + n]));
          }
        printf("{\"test\":\"t11_swizzle_window\",\"RB\":%d,\"N\":%d,\"a0\":%d,\"maxerr\":%.3g,\"pass\":%s}\n", RB, N,
               a0, e, e < 1e-3 ? "true" : "false");
      }
    cudaFree(dA), cudaFree(dB), cudaFree(dD);
  }
}

// SS throughput with RB-swizzled operands: M=128, N, K = RB/2 per "block" (RB/32 MMAs of K=16)
__global__ void __launch_bounds__(128, 1) k_thr_swz(int N, int RB, int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  int w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  fence_async_smem();
  if (w == 0) tmem_alloc<512>(&tslot), tmem_relinquish();
  if (threadIdx.x == 32) mbar_init(&bar, 1), fence_mbar_init();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    uint32_t idesc = idesc_f32acc(1, 128, N);
    const int nk = RB / 32;
    const uint32_t sbo = 8 * RB;
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
      for (int k = 0; k < nk; ++k) {
        uint32_t sa = smem_u32(smem) + (it & 7) * RB * 3 + k * 32;     // shifting A windows, as in the convs
        uint32_t sb = smem_u32(smem) + 32768 + k * 32;
        umma_f16_ss(tb, smem_desc(sa, 16, sbo, layout_of(RB)), smem_desc(sb, 16, sbo, layout_of(RB)), idesc, 1);
      }
    umma_commit(&bar);
    wait_bounded(&bar, 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (w == 0) tmem_dealloc<512>(tb);
}

static void t12(int nsm) {
  unsigned long long* dc;
  CK(cudaMalloc(&dc, nsm * 8));
  CK(cudaFuncSetAttribute(k_thr_swz, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024));
  for (int RB : {32, 64, 128})
    for (int N : {16, 32, 64, 128, 256}) {
      const int nk = RB / 32;
      int iters = 2048 * 256 / N / nk;
      k_thr_swz<<<nsm, 128, 65536 + 1024>>>(N, RB, 16, dc);
      k_thr_swz<<<nsm, 128, 65536 + 1024>>>(N, RB, iters, dc);
      if (check_err("t12")) return;
      std::vector<unsigned long long> hc(nsm);
      CK(cudaMemcpy(hc.data(), dc, nsm * 8, cudaMemcpyDeviceToHost));
      double cmax = 0;
      for (int i = 0; i < nsm; ++i) cmax = fmax(cmax, (double)hc[i]);
      double mmas = (double)iters * nk;
      printf("{\"test\":\"t12_ss_throughput\",\"RB\":%d,\"N\":%d,\"cyc_per_mma\":%.2f,\"floor_cyc\":%.1f,"
             "\"smem_B_per_clk\":%.1f}\n", RB, N, cmax / mmas, 128.0 * N / 256.0, (128.0 * 32 + N * 32.0) / (cmax / mmas));
    }
  cudaFree(dc);
}

// t13: A = aligned SW128 weights (M=128), B = RB-swizzled activations at shifted windows (the conv mapping)
__global__ void __launch_bounds__(128, 1) k_thr_b(int N, int RB, int iters, int shift, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  int w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  fence_async_smem();
  if (w == 0) tmem_alloc<512>(&tslot), tmem_relinquish();
  if (threadIdx.x == 32) mbar_init(&bar, 1), fence_mbar_init();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    uint32_t idesc = idesc_f32acc(1, 128, N);
    const uint32_t sbo = 8 * RB;
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int k = it & 3;
      uint32_t sa = smem_u32(smem) + k * 32;
      uint32_t sb = smem_u32(smem) + 16384 + (shift ? (it % 11) * 74 * RB : 0) + (k % (RB / 32)) * 32;
      umma_f16_ss(tb, smem_desc(sa, 16, 1024, 2), smem_desc(sb, 16, sbo, layout_of(RB)), idesc, 1);
    }
    umma_commit(&bar);
    wait_bounded(&bar, 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (w == 0) tmem_dealloc<512>(tb);
}
static void t13(int nsm) {
  unsigned long long* dc;
  CK(cudaMalloc(&dc, nsm * 8));
  CK(cudaFuncSetAttribute(k_thr_b, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304 + 1024));
  for (int RB : {32, 64, 128})
    for (int N : {64, 128, 256})
      for (int shift : {0, 1}) {
        if (16384 + 10 * 74 * RB + N * RB > 98304) continue;
        int iters = 4096 * 256 / N;
        k_thr_b<<<nsm, 128, 98304 + 1024>>>(N, RB, 16, shift, dc);
        k_thr_b<<<nsm, 128, 98304 + 1024>>>(N, RB, iters, shift, dc);
        if (check_err("t13")) return;
        std::vector<unsigned long long> hc(nsm);
        CK(cudaMemcpy(hc.data(), dc, nsm * 8, cudaMemcpyDeviceToHost));
        double cmax = 0;
        for (int i = 0; i < nsm; ++i) cmax = fmax(cmax, (double)hc[i]);
        printf("{\"test\":\"t13_B_swizzle_throughput\",\"RB\":%d,\"N\":%d,\"shift\":%d,\"cyc_per_mma\":%.2f,"
               "\"floor_cyc\":%.1f}\n", RB, N, shift, cmax / iters, 128.0 * N / 256.0);
      }
  cudaFree(dc);
}

// t14: like t13 with `nacc` accumulators interleaved (is the per-MMA floor a D-dependency latency?)
__global__ void __launch_bounds__(128, 1) k_thr_acc(int N, int RB, int iters, int nacc, int mode,
                                                     unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  int w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 200704 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  fence_async_smem();
  if (w == 0) tmem_alloc<512>(&tslot), tmem_relinquish();
  if (threadIdx.x == 32) mbar_init(&bar, 1), fence_mbar_init();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    uint32_t idesc = idesc_f32acc(1, 128, N);
    const uint32_t sbo = 8 * RB;
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem) + 16384;
    unsigned long long t0 = clock64();
    int sh = 0;
    for (int it = 0; it < iters; ++it) {
      const int k = it & 3;
      const uint32_t sa = a0 + k * 32;
      const uint32_t sb = b0 + (mode ? sh * RB : 0) + (k & (RB / 32 - 1)) * 32;
      if (++sh == 11 * 74) sh = 0;
      const uint32_t d = tb + (uint32_t)((it % nacc) * N);
      umma_f16_ss(d, smem_desc(sa, 16, 1024, 2), smem_desc(sb, 16, sbo, layout_of(RB)), idesc, 1);
    }
    umma_commit(&bar);
    wait_bounded(&bar, 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (w == 0) tmem_dealloc<512>(tb);
}
static void t14(int nsm) {
  unsigned long long* dc;
  CK(cudaMalloc(&dc, nsm * 8));
  const int SM = 200704;
  CK(cudaFuncSetAttribute(k_thr_acc, cudaFuncAttributeMaxDynamicSharedMemorySize, SM + 1024));
  for (int RB : {32, 64, 128})
    for (int N : {32, 64, 128, 256})
      for (int nacc : {1, 2, 4})
        for (int mode : {0, 1}) {
          if (nacc * N > 512) continue;
          if (16384 + 11 * 74 * RB + 256 * RB > SM) continue;
          int iters = 4096 * 256 / N;
          k_thr_acc<<<nsm, 128, SM + 1024>>>(N, RB, 16, nacc, mode, dc);
          k_thr_acc<<<nsm, 128, SM + 1024>>>(N, RB, iters, nacc, mode, dc);
          if (check_err("t14")) return;
          std::vector<unsigned long long> hc(nsm);
          CK(cudaMemcpy(hc.data(), dc, nsm * 8, cudaMemcpyDeviceToHost));
          double cmax = 0;
          for (int i = 0; i < nsm; ++i) cmax = fmax(cmax, (double)hc[i]);
          printf("{\"test\":\"t14\",\"RB\":%d,\"N\":%d,\"nacc\":%d,\"shift\":%d,\"cyc_per_mma\":%.2f,\"floor\":%.0f}\n",
                 RB, N, nacc, mode, cmax / iters, 128.0 * N / 256.0);
        }
  cudaFree(dc);
}

// t15: register layout of tcgen05.ld.16x256b (x1 and x2) and 16x64b: TMEM cell (lane, col) = lane*1000 + col
__global__ void k_t15(float* out) {
  __shared__ uint32_t tslot;
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (w == 0) tmem_alloc<512>(&tslot), tmem_relinquish();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tb = tslot;
  for (int c = 0; c < 64; c += 16) {
    uint32_t r[16];
    for (int j = 0; j < 16; ++j) r[j] = __float_as_uint((float)((w * 32 + l) * 1000 + c + j));
    tmem_st16(tb + ((uint32_t)(w * 32) << 16) + c, r);
  }
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (w == 0) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(tb));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 4; ++j) out[l * 16 + j] = __uint_as_float(r[j]);
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tb + (16u << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) out[l * 16 + 4 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (w == 0) tmem_dealloc<512>(tb);
}
static void t15() {
  float* d;
  CK(cudaMalloc(&d, 32 * 16 * 4));
  k_t15<<<1, 128>>>(d);
  if (check_err("t15")) return;
  std::vector<float> h(32 * 16);
  CK(cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost));
  for (int t = 0; t < 32; ++t) {
    printf("{\"test\":\"t15\",\"thread\":%d,\"x1_lane0\":[", t);
    for (int j = 0; j < 4; ++j) printf("%s%.0f", j ? "," : "", h[t * 16 + j]);
    printf("],\"x2_lane16\":[");
    for (int j = 0; j < 8; ++j) printf("%s%.0f", j ? "," : "", h[t * 16 + 4 + j]);
    printf("]}\n");
  }
  cudaFree(d);
}

// ------------------------------------------------------------------------ t16: disable-output-lane
// tcgen05.mma's optional disable-output-lane operand (4 x 32-bit masks for cta_group::1, one bit per TMEM lane):
// which lanes of D does an MMA leave untouched, with and without enable-input-d?  TMEM is pre-filled with -1,
// A = ones in K column 1, B[n] = n + 1 in K column 1, so an enabled lane reads n + 1 (overwrite) or n (accumulate).
__device__ __forceinline__ void umma_f16_ss_dol(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc,
                                                uint32_t m0, uint32_t m1, uint32_t m2, uint32_t m3) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(m0), "r"(m1), "r"(m2), "r"(m3)
      : "memory");
}
__global__ void k_dol(const __nv_bfloat16* A, const __nv_bfloat16* B, int N, uint32_t acc, uint32_t m0, uint32_t m1,
                      uint32_t m2, uint32_t m3, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + 32768;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  int w = threadIdx.x >> 5;
  st_sw128(sA, A, 128);
  st_sw128(sB, B, 320);
  fence_async_smem();
  if (w == 0) tmem_alloc<512>(&tslot), tmem_relinquish();
  if (threadIdx.x == 32) mbar_init(&bar, 1), fence_mbar_init();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tb = tslot;
  if (w < 4) {
    uint32_t r[16];
    for (int j = 0; j < 16; ++j) r[j] = __float_as_uint(-1.0f);
    for (int c = 0; c < 512; c += 16) tmem_st16(tb + ((uint32_t)(w * 32) << 16) + c, r);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    uint32_t idesc = idesc_f32acc(1, 128, N);
    uint64_t ad = smem_desc(smem_u32(sA), 16, 1024, kSwizzle128B);
    uint64_t bd = smem_desc(smem_u32(sB), 16, 1024, kSwizzle128B);
    umma_f16_ss_dol(tb, ad, bd, idesc, acc, m0, m1, m2, m3);
    umma_commit(&bar);
    wait_bounded(&bar, 0);
  }
  __syncthreads();
  tc_fence_after();
  dump_tmem(tb, out, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (w == 0) tmem_dealloc<512>(tb);
}

static void t16() {
  std::vector<__nv_bfloat16> A(128 * 64), B(320 * 64);
  for (auto& v : A) v = __float2bfloat16(0.f);
  for (auto& v : B) v = __float2bfloat16(0.f);
  for (int m = 0; m < 128; ++m) A[m * 64 + 1] = __float2bfloat16(1.f);
  for (int n = 0; n < 320; ++n) B[n * 64 + 1] = __float2bfloat16((float)(n + 1));
  __nv_bfloat16 *dA = dup(A), *dB = dup(B);
  float* dD;
  CK(cudaMalloc(&dD, 128 * 512 * 4));
  CK(cudaFuncSetAttribute(k_dol, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304));
  std::vector<float> D(128 * 512);
  struct S { uint32_t acc, m[4]; const char* name; };
  std::vector<S> ss = {
      {0, {0, 0, 0, 0}, "overwrite_mask0"},
      {0, {0x0000F800u, 0, 0, 0}, "overwrite_disable_lanes11to15"},
      {1, {0x0000F800u, 0, 0, 0}, "accumulate_disable_lanes11to15"},
      {0, {0xFFFF07FFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu}, "overwrite_only_lanes11to15"},
      {1, {0, 0x00000001u, 0, 0x80000000u}, "accumulate_disable_lane32_and_127"},
  };
  const int N = 64;
  for (auto s : ss) {
    k_dol<<<1, 128, 98304>>>(dA, dB, N, s.acc, s.m[0], s.m[1], s.m[2], s.m[3], dD);
    if (check_err("t16")) return;
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    // classify every lane by its columns 0..N-1: 'k' kept (-1), 'w' written (n + 1), 'a' accumulated (n), '?' other
    std::string cls(128, '?');
    int exact = 1;
    for (int l = 0; l < 128; ++l) {
      int k = 1, w = 1, a = 1;
      for (int c = 0; c < N; ++c) {
        const float v = D[l * 512 + c];
        k &= v == -1.f, w &= v == (float)(c + 1), a &= v == (float)c;
      }
      cls[l] = k ? 'k' : (w ? 'w' : (a ? 'a' : '?'));
      const bool dis = (s.m[l >> 5] >> (l & 31)) & 1u;
      const char want = dis ? 'k' : (s.acc ? 'a' : 'w');
      exact &= cls[l] == want;
    }
    int beyond = 1;   // columns >= N untouched
    for (int l = 0; l < 128; ++l)
      for (int c = N; c < 512; ++c) beyond &= D[l * 512 + c] == -1.f;
    printf("{\"test\":\"t16_%s\",\"acc\":%u,\"masks\":[%u,%u,%u,%u],\"lanes\":\"%s\",\"as_expected\":%d,"
           "\"cols_beyond_N_untouched\":%d}\n", s.name, s.acc, s.m[0], s.m[1], s.m[2], s.m[3], cls.c_str(), exact, beyond);
  }
  cudaFree(dA), cudaFree(dB), cudaFree(dD);
}


int main(int argc, char** argv) {
  int dev = 0, nsm = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, dev));
  printf("{\"device\":\"%s\",\"sm\":%d,\"cc\":\"%d.%d\",\"l2\":%d}\n", p.name, nsm, p.major, p.minor, p.l2CacheSize);
  std::string which = argc > 1 ? argv[1] : "all";
  auto on = [&](const char* t) { return which == "all" || which.find(t) != std::string::npos; };
  if (on("t1")) t1();
  if (on("t2") || on("t3") || on("t4")) t234();
  if (on("t5")) t5();
  if (on("t6")) t6(nsm);
  if (on("t7")) t7(nsm);
  if (on("t9")) t9(nsm);
  if (on("t10")) t10();
  if (on("t11")) t11();
  if (on("t12")) t12(nsm);
  if (on("t13")) t13(nsm);
  if (on("t14")) t14(nsm);
  if (on("t15")) t15();
  if (on("t16")) t16();
  return 0;
}
