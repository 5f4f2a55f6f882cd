// L2 -> shared-memory bulk-copy throughput per SM, the way conv2 streams its weights: every CTA (one per SM)
// cycles through the same L2-resident 528-KB buffer in copies of CH bytes, NS copies in flight (a ring of NS slots
// with mbarrier completion, a slot re-armed as soon as its copy landed).  Reports bytes / SM clock and copies /
// 1000 clocks per SM: is the stream bound by bytes or by the number of copies?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/scratch/l2_bulk_probe tools/scratch/l2_bulk_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NS>
__global__ void k_stream(const uint8_t* src, uint32_t src_bytes, uint32_t ch, int copies, long long* cyc) {
  // one producer thread per warp (lane 0), each with its own ring of NS slots (blockDim.x / 32 producers)
  extern __shared__ __align__(1024) uint8_t smraw[];
  __shared__ uint64_t bars[4][NS];
  if ((threadIdx.x & 31) != 0) return;
  const int w = threadIdx.x >> 5;
  uint64_t* bar = bars[w];
  uint8_t* sm = smraw + (size_t)w * NS * ch;
  for (int i = 0; i < NS; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t ph[NS] = {};
  const long long t0 = clock64();
  uint32_t off = (blockIdx.x * 4096u) % src_bytes;
  for (int k = 0; k < copies; ++k) {
    const int s = k % NS;
    const uint32_t b = su32(&bar[s]);
    if (k >= NS) {
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(b), "r"(ph[s]) : "memory");
      ph[s] ^= 1;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(ch) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(sm + s * ch)), "l"(src + off), "r"(ch), "r"(b) : "memory");
    off += ch;
    if (off + ch > src_bytes) off = 0;
  }
  for (int s = 0; s < NS; ++s) {
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(su32(&bar[s])), "r"(ph[s]) : "memory");
  }
  if (w == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint32_t SRC = 528 * 1024;
  uint8_t* src;
  long long* cyc;
  cudaMalloc(&src, SRC);
  cudaMemset(src, 1, SRC);
  cudaMalloc(&cyc, sms * sizeof(long long));
  long long h[1024];
  auto run = [&](auto kern, int ns, uint32_t ch, int nw = 1) {
    const int smem = ns * ch * nw;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int copies = (int)((64ull << 20) / ch);   // 64 MB per SM
    for (int rep = 0; rep < 2; ++rep) kern<<<sms, 32 * nw, smem>>>(src, SRC, ch, copies, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0, sum = 0;
    for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx, sum += h[i];
    const double avg = (double)sum / sms;
    printf("{\"copy_KB\": %u, \"producers\": %d, \"in_flight_each\": %d, \"bytes_per_clk_per_sm\": %.1f, "
           "\"copies_per_kclk\": %.2f, \"err\": \"%s\"}\n", ch / 1024, nw, ns, (double)copies * ch * nw / avg,
           copies * nw / avg * 1000.0,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (uint32_t ch : {4096u, 8192u, 16384u}) {
    run(k_stream<4>, 4, ch, 1);
    run(k_stream<4>, 4, ch, 2);
    run(k_stream<4>, 4, ch, 3);
  }
  run(k_stream<2>, 2, 32768u, 1);
  run(k_stream<2>, 2, 32768u, 2);
  return 0;
}
