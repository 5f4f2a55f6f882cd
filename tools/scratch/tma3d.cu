// standalone check: 3-D bf16 TMA box with out-of-bounds coordinates (conv1 strip load)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>
#include "../../paper_1701_03891_b200/csrc/sm100.cuh"
using namespace di;
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap m, int bw, int bh, int c0, int r0, uint16_t* out) {
  extern __shared__ __align__(128) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, bw * bh * 2);
    tma_load_3d(sm, &m, &bar, c0, r0, 1);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < bw * bh; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(sm)[i];
}
int main() {
  int n1 = 16, n2 = 16, B = 4, bw = 32, bh = 26;
  std::vector<uint16_t> h(B * n1 * n2);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (uint16_t)(i + 1);
  uint16_t *d, *o;
  cudaMalloc(&d, h.size() * 2); cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  cudaMalloc(&o, bw * bh * 2);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)n2, (cuuint64_t)n1, (cuuint64_t)B};
  cuuint64_t str[2] = {(cuuint64_t)n2 * 2, (cuuint64_t)n1 * n2 * 2};
  cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1}, es[3] = {1, 1, 1};
  CUresult r = ((Enc)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  int c0 = getenv("C0") ? atoi(getenv("C0")) : -5;
  k<<<1, 128, bw * bh * 2 + 1024>>>(m, bw, bh, c0, c0, o);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<uint16_t> ho(bw * bh);
  cudaMemcpy(ho.data(), o, ho.size() * 2, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int rr = 0; rr < bh; ++rr) for (int cc = 0; cc < bw; ++cc) {
    int gy = rr + (getenv("C0") ? atoi(getenv("C0")) : -5), gx = cc + (getenv("C0") ? atoi(getenv("C0")) : -5);
    uint16_t want = (gy >= 0 && gy < n1 && gx >= 0 && gx < n2) ? h[(1 * n1 + gy) * n2 + gx] : 0;
    bad += ho[rr * bw + cc] != want;
  }
  printf("bad %d\n", bad);
  return 0;
}
