// tools/scratch/swz_rate.cu -- probe: SS UMMA (kind::f16, M = 128, K-major) cycles per MMA vs the operand swizzle
// (128 / 64 / 32-B rows) and N.  Not part of the product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/scratch/swz_rate tools/scratch/swz_rate.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include "../../paper_1701_03891_b200/csrc/sm100.cuh"
using namespace di;

template <int ROWB, int N, int NWIN>
__global__ void __launch_bounds__(128, 1) k_rate(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 196608 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  fence_async_smem();
  if (w == 0) tmem_alloc<512>(&tslot), tmem_relinquish();
  if (threadIdx.x == 32) mbar_init(&bar, 1), fence_mbar_init();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t swz = ROWB == 128 ? kSwizzle128B : (ROWB == 64 ? kSwizzle64B : kSwizzle32B);
    constexpr uint32_t sbo = 8 * ROWB;
    const uint32_t idesc = idesc_f32acc(1, 128, N);
    // A windows start at different 1-KB-aligned offsets (like the conv3 stack / the conv2 weight ring);
    // B windows at different rows of a strip (like the tap shifts)
    const uint64_t a0 = smem_desc(smem_u32(smem), 16, sbo, swz);
    const uint64_t b0 = smem_desc(smem_u32(smem) + 65536, 16, sbo, swz);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < NWIN; ++k) {
        const uint64_t ad = a0 + (uint64_t)((k * 1024) >> 4);
        const uint64_t bd = b0 + (uint64_t)((k * 5 * ROWB) >> 4);
#pragma unroll
        for (int kk = 0; kk < ROWB / 32; ++kk)
          umma_f16_ss(tb + (k & 1) * 256, ad + 2 * kk, bd + 2 * kk, idesc, 1);
      }
    }
    umma_commit(&bar);
    while (!mbar_try_wait(&bar, 0)) {}
    cyc[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (w == 0) tmem_dealloc<512>(tb);
}

template <int ROWB, int N>
static void run(int nsm, unsigned long long* dc) {
  constexpr int NWIN = 8;
  auto k = k_rate<ROWB, N, NWIN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608);
  const int iters = 2048;
  k<<<nsm, 128, 196608>>>(16, dc);
  k<<<nsm, 128, 196608>>>(iters, dc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
  std::vector<unsigned long long> h(nsm);
  cudaMemcpy(h.data(), dc, nsm * 8, cudaMemcpyDeviceToHost);
  double cmax = 0;
  for (auto v : h) cmax = cmax > v ? cmax : (double)v;
  const double mmas = (double)iters * NWIN * (ROWB / 32);
  const double cpm = cmax / mmas, ideal = N / 2.0;
  printf("{\"rowB\":%d,\"N\":%d,\"cyc_per_mma\":%.1f,\"ideal\":%.0f,\"frac\":%.3f,\"operand_B_per_clk\":%.1f}\n", ROWB, N,
         cpm, ideal, ideal / cpm, (128 * 32 + N * 32) / cpm);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* dc;
  cudaMalloc(&dc, nsm * 8);
  run<128, 256>(nsm, dc); run<64, 256>(nsm, dc); run<32, 256>(nsm, dc);
  run<128, 160>(nsm, dc); run<64, 160>(nsm, dc);
  run<128, 80>(nsm, dc); run<64, 80>(nsm, dc); run<32, 80>(nsm, dc);
  run<128, 64>(nsm, dc); run<64, 64>(nsm, dc);
  return 0;
}
