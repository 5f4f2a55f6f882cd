// tools/scratch/ffma2_rate.cu -- probe: FFMA vs packed FFMA2 (fma.rn.f32x2) throughput per SM on sm_100a.
// Not part of the product.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/scratch/ffma2_rate tools/scratch/ffma2_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
template <bool PACKED>
__global__ void k(float* out, int iters, float s) {
  float a[16];
  unsigned long long p[8];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
#pragma unroll
  for (int i = 0; i < 8; ++i) { float2 t = make_float2(a[2 * i], a[2 * i + 1]); p[i] = *reinterpret_cast<unsigned long long*>(&t); }
  float2 ss = make_float2(s, s);
  unsigned long long sp = *reinterpret_cast<unsigned long long*>(&ss);
  float2 cc = make_float2(0.5f, 0.25f);
  unsigned long long cp = *reinterpret_cast<unsigned long long*>(&cc);
  for (int it = 0; it < iters; ++it) {
    if (PACKED) {
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(sp), "l"(cp));
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(s), "f"(0.5f + i));
    }
  }
  float r = 0;
  if (PACKED) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { float2 t = *reinterpret_cast<float2*>(&p[i]); r += t.x + t.y; }
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) r += a[i];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* o;
  cudaMalloc(&o, nsm * 8 * 1024 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep)
    for (int packed = 0; packed < 2; ++packed) {
      for (int warps : {8, 16, 32}) {
        const int blocks = nsm * 4, threads = warps * 32 / 4;
        if (packed) k<true><<<blocks, threads>>>(o, 10, 0.999f); else k<false><<<blocks, threads>>>(o, 10, 0.999f);
        cudaEventRecord(e0);
        if (packed) k<true><<<blocks, threads>>>(o, iters, 0.999f); else k<false><<<blocks, threads>>>(o, iters, 0.999f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fmas = (double)blocks * threads * iters * 16;
        if (rep == 1) printf("{\"packed\":%d,\"warps_per_sm\":%d,\"tflops\":%.1f}\n", packed, warps, 2 * fmas / (ms * 1e-3) / 1e12);
      }
    }
  return 0;
}
