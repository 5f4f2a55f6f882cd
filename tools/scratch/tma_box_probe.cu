// conv3's strip feed in isolation: every CTA (one per SM) streams h2 rows of image pairs into a 12-slot shared-memory
// ring, as k_conv3_r4's producer does -- (a) one 4-D TMA box per strip row (32 channels x 80 columns with 5 / 11
// out-of-bounds zero columns x 2 images x 1 row, 10 KB), (b) the same rows as two plain 1-D bulk copies of the 4-KB
// in-bounds image rows -- over the whole 1.07-GB h2 of the lowrate batch.  Reports GB/s and clocks per row per SM:
// is the 4-D box feed slower than the HBM read floor?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/scratch/tma_box_probe tools/scratch/tma_box_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int NSL = 12, N1 = 64, N2 = 64, C = 32, PP = 80;

__device__ __forceinline__ void wait_bar(uint32_t b, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(b), "r"(ph) : "memory");
}

template <bool BOX>
__global__ void k_feed(const __grid_constant__ CUtensorMap tm, const uint8_t* h2, int pairs, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[NSL];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < NSL; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint32_t rowb = 2 * PP * 64;
  uint32_t ph[NSL] = {};
  int k = 0;
  const long long t0 = clock64();
  for (int p = blockIdx.x; p < pairs; p += gridDim.x)
    for (int s = 0; s < N1; ++s, ++k) {
      const int sl = k % NSL;
      const uint32_t b = su32(&bar[sl]);
      if (k >= NSL) wait_bar(b, ph[sl]), ph[sl] ^= 1;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(BOX ? rowb : 2u * N2 * C * 2)
                   : "memory");
      if (BOX) {
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
            "[%6];" ::"r"(su32(sm + sl * rowb)), "l"(&tm), "r"(0), "r"(-5), "r"(2 * p), "r"(s), "r"(b) : "memory");
      } else {
        for (int i = 0; i < 2; ++i) {
          const uint8_t* src = h2 + (((size_t)(2 * p + i) * N1 + s) * N2) * C * 2;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(su32(sm + sl * rowb + i * PP * 64 + 5 * 64)), "l"(src), "r"(N2 * C * 2), "r"(b) : "memory");
        }
      }
    }
  for (int i = 0; i < NSL && i < k; ++i) wait_bar(su32(&bar[i]), ph[i]);
  cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int B = 4096, pairs = B / 2;
  const size_t bytes = (size_t)B * N1 * N2 * C * 2;
  uint8_t* h2;
  long long* cyc;
  cudaMalloc(&h2, bytes);
  cudaMemset(h2, 0, bytes);
  cudaMalloc(&cyc, sms * sizeof(long long));
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  CUtensorMap tm;
  // dims (channel, column, image, row) as in k_conv3_r4: the box lands as [row][image][column][channel]
  cuuint64_t dims[4] = {C, N2, (cuuint64_t)B, N1};
  cuuint64_t strides[3] = {C * 2, (cuuint64_t)N1 * N2 * C * 2, (cuuint64_t)N2 * C * 2};
  cuuint32_t box[4] = {C, PP, 2, 1}, es[4] = {1, 1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, h2, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  const int smem = NSL * 2 * PP * 64;
  cudaFuncSetAttribute(k_feed<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_feed<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long h[1024];
  for (int mode = 0; mode < 2; ++mode)
    for (int rep = 0; rep < 3; ++rep) {
      cudaEvent_t a, b;
      cudaEventCreate(&a), cudaEventCreate(&b);
      cudaEventRecord(a);
      if (mode == 0) k_feed<true><<<sms, 32, smem>>>(tm, h2, pairs, cyc);
      else k_feed<false><<<sms, 32, smem>>>(tm, h2, pairs, cyc);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      cudaMemcpy(h, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
      const double rows_per_sm = (double)pairs / sms * N1;
      printf("{\"feed\": \"%s\", \"ms\": %.4f, \"GBs_of_h2\": %.0f, \"clocks_per_row_max_sm\": %.0f, \"err\": \"%s\"}\n",
             mode == 0 ? "4-D TMA box per row (conv3)" : "2 x 1-D bulk copies per row", ms, bytes / ms / 1e6,
             mx / rows_per_sm, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
