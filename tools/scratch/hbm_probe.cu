// HBM write-only / read-only floors for conv1 (writes h1, 2.15 GB) and conv3 (reads h2, 1.07 GB) on this B200:
// plain 16-B vector stores / loads (grid-stride, CTAs = k x SMs) and bulk copies (cp.async.bulk) between shared
// memory and global memory, the path conv1's TMA-store epilogue and conv3's TMA loads use.  CUDA events, best of 10.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/scratch/hbm_probe tools/scratch/hbm_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void k_store_v4(uint4* p, size_t n16) {
  const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}

__global__ void k_load_v4(const uint4* p, size_t n16, unsigned* sink) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldcs(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

// one thread per CTA issues bulk stores of CH bytes from shared memory, keeping DEPTH groups in flight
template <int CH, int DEPTH>
__global__ void k_bulk_store(uint8_t* p, size_t nbytes) {
  extern __shared__ __align__(128) uint8_t sm[];
  for (int i = threadIdx.x; i < CH / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
  for (size_t off = (size_t)blockIdx.x * CH; off < nbytes; off += (size_t)gridDim.x * CH) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p + off), "r"(s), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(DEPTH) : "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// one thread per CTA issues bulk loads of CH bytes into a ring of NS shared-memory slots (mbarrier completion)
template <int CH, int NS>
__global__ void k_bulk_load(const uint8_t* p, size_t nbytes, unsigned* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar[NS];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < NS; ++i) {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[i]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
  uint32_t ph[NS] = {};
  int k = 0;
  for (size_t off = (size_t)blockIdx.x * CH; off < nbytes; off += (size_t)gridDim.x * CH, ++k) {
    const int sl = k % NS;
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[sl]);
    if (k >= NS) {   // wait for the slot's previous load
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(b), "r"(ph[sl]) : "memory");
      ph[sl] ^= 1;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(s + sl * CH), "l"(p + off), "r"(CH), "r"(b) : "memory");
  }
  for (int sl = 0; sl < NS && sl < k; ++sl) {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[sl]);
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(b), "r"(ph[sl]) : "memory");
  }
  if (sm[0] == 0x5a && sm[1] == 0xa5) sink[0] = 1;
}

template <typename F>
static float best(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a), cudaEventCreate(&b);
  float bestms = 1e30f;
  for (int r = 0; r < 12; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r >= 2 && ms < bestms) bestms = ms;
  }
  return bestms;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t W = 2ull * 4096 * 4096 * 64;   // h1 bytes (bf16, 64 ch, 4096 images of 64x64)
  const size_t R = W / 2;                       // h2 bytes
  uint8_t* buf;
  unsigned* sink;
  CK(cudaMalloc(&buf, W));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(buf, 1, W));
  for (int k : {1, 2, 4, 8}) {
    const float ms = best([&] { k_store_v4<<<sms * k, 512>>>(reinterpret_cast<uint4*>(buf), W / 16); });
    printf("{\"probe\": \"store_v4\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"GBs\": %.1f}\n", k, ms, W / ms / 1e6);
  }
  for (int k : {1, 2, 4, 8}) {
    const float ms = best([&] { k_load_v4<<<sms * k, 512>>>(reinterpret_cast<const uint4*>(buf), R / 16, sink); });
    printf("{\"probe\": \"load_v4\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"GBs\": %.1f}\n", k, ms, R / ms / 1e6);
  }
  CK(cudaFuncSetAttribute(k_bulk_store<32768, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
  CK(cudaFuncSetAttribute(k_bulk_store<16384, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
  for (int k : {1, 2, 4}) {
    float ms = best([&] { k_bulk_store<32768, 4><<<sms * k, 128, 32768>>>(buf, W); });
    printf("{\"probe\": \"bulk_store_32K_depth4\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"GBs\": %.1f}\n", k, ms, W / ms / 1e6);
    ms = best([&] { k_bulk_store<16384, 8><<<sms * k, 128, 16384>>>(buf, W); });
    printf("{\"probe\": \"bulk_store_16K_depth8\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"GBs\": %.1f}\n", k, ms, W / ms / 1e6);
  }
  CK(cudaFuncSetAttribute(k_bulk_load<16384, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384));
  CK(cudaFuncSetAttribute(k_bulk_load<10240, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 10240));
  for (int k : {1}) {
    float ms = best([&] { k_bulk_load<16384, 8><<<sms * k, 32, 8 * 16384>>>(buf, R, sink); });
    printf("{\"probe\": \"bulk_load_16K_ring8\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"GBs\": %.1f}\n", k, ms, R / ms / 1e6);
    ms = best([&] { k_bulk_load<10240, 12><<<sms * k, 32, 12 * 10240>>>(buf, R, sink); });
    printf("{\"probe\": \"bulk_load_10K_ring12 (conv3 rows)\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"GBs\": %.1f}\n", k, ms, R / ms / 1e6);
  }
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return 0;
}
