// k_proxy.cu -- stage 0, the lifting layer: x_tilde_b = Phi^T y_b for a batch,
// written straight into the row-major n1 x n2 image layout that conv layer 1 reads.
//
// As one batched GEMM  X_tilde[B][N] = Y[B][M] * Phi[M][N].
//   bf16 / tf32: tcgen05 UMMA, D tile 128 (images) x 256 (pixels) in TMEM, A = Y tile and B = Phi^T tile
//         staged by TMA (SWIZZLE_128B, K-major; the K tail M..Kpad is zero-filled by the packing of Phi^T
//         and by TMA out-of-bounds fill of Y), 4-stage mbarrier pipeline, warp-specialised
//         (warp 0 TMA producer, warp 1 MMA issuer, warps 0-3 epilogue).
//   fp32: SIMT FFMA tiled GEMM with two-level (per-K-tile, then total) accumulation for the 1e-5 parity bar.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "kernels.cuh"
#define DI_TU_ID 1
#include "sm100.cuh"

namespace di {

namespace {
constexpr int PX_BM = 128;      // images per tile (UMMA M)
constexpr int PX_BN = 256;      // pixels per tile (UMMA N); BN = 224 for the lifting layer when it fills the waves better
constexpr int PX_STAGES = 4;
constexpr int PX2_STAGES = 4;   // k_proxy_pair: 4 x (16 KB + BN x 128 B)
}  // namespace

// ELT: 2 = bf16 (kind::f16, K=16 per MMA), 4 = fp32 storage with kind::tf32 (K=8 per MMA).
// OF32: fp32 output even for bf16 operands (row-sharded partial proxies, summed across ranks before rounding)
// MB: 128-image batch tiles per CTA.  MB = 2 gives each Phi^T K-block (32 KB) to two accumulators (TMEM 2 x 256
// columns): per 1024 MMA cycles the SM ingests 64 KB instead of 2 x 48 KB -- what bounds the GEMM when Phi streams
// from HBM (Stress: 2.15 GB of Phi, each CTA's L2 -> SM ingest at ~94 B/clk with MB = 1).  3 stages of 64 KB.
template <int ELT, bool OF32 = (ELT == 4), int MB = 1, int BN = PX_BN>
__global__ void __launch_bounds__(128, 1)
    k_proxy_tc(const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmPt, int batch,
               int N, int kblocks, void* __restrict__ xt, ProxyScatter sc, int bblk) {
  constexpr int KB_ELEMS = 128 / ELT;                       // K elements per 128-B swizzle row
  constexpr uint32_t A_BYTES = MB * PX_BM * 128, B_BYTES = BN * 128;
  constexpr uint32_t STAGE = A_BYTES + B_BYTES;
  constexpr int NST = MB == 1 ? PX_STAGES : 3;
  constexpr int K_PER_MMA = 32 / ELT;                        // 16 (bf16) or 8 (tf32)
  constexpr int MMAS_PER_KB = KB_ELEMS / K_PER_MMA;          // 4
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ uint64_t full[NST], empty[NST], tfull;
  __shared__ uint32_t tslot;

  const int warp = warp_id(), lane = lane_id();
  const int nbt = (batch + PX_BM * MB - 1) / (PX_BM * MB);
  const int bt = blockIdx.x % nbt, nt = blockIdx.x / nbt;   // consecutive CTAs share one Phi^T slice (L2)
  const int b0 = bt * PX_BM * MB, n0 = nt * BN;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmY);
    tma_prefetch_desc(&tmPt);
    for (int s = 0; s < NST; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    mbar_init(&tfull, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<256 * MB>(&tslot), tmem_relinquish();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  griddep_wait();                 // the preceding grid's outputs (PDL: only the prologue above overlapped it)
  griddep_launch_dependents();

  if (warp == 0 && lane == 0) {  // ---------------- TMA producer
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % NST;
      if (kb >= NST) mbar_wait(&empty[s], ((kb / NST) - 1) & 1);
      uint8_t* sa = smem + s * STAGE;
      mbar_arrive_expect_tx(&full[s], STAGE);
#pragma unroll
      for (int h = 0; h < MB; ++h) tma_load_2d(sa + h * PX_BM * 128, &tmY, &full[s], kb * KB_ELEMS, b0 + h * PX_BM);
      if (bblk)   // tile-blocked Phi^T: block (n-tile, kb) is one contiguous 32 KB
        tma_load_3d(sa + A_BYTES, &tmPt, &full[s], 0, 0, nt * kblocks + kb);
      else
        tma_load_2d(sa + A_BYTES, &tmPt, &full[s], kb * KB_ELEMS, n0);
    }
  } else if (warp == 1 && lane == 0) {  // ---------------- MMA issuer
    constexpr uint32_t idesc = idesc_f32acc(ELT == 2 ? 1 : 2, PX_BM, BN);
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % NST;
      mbar_wait(&full[s], (kb / NST) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * STAGE), sb = sa + A_BYTES;
#pragma unroll
      for (int k = 0; k < MMAS_PER_KB; ++k) {
        const uint64_t bd = smem_desc(sb + k * 32, 16, 1024, kSwizzle128B);
#pragma unroll
        for (int h = 0; h < MB; ++h) {
          const uint64_t ad = smem_desc(sa + h * PX_BM * 128 + k * 32, 16, 1024, kSwizzle128B);
          if (ELT == 2)
            umma_f16_ss(tmem + h * 256, ad, bd, idesc, (kb | k) != 0);
          else
            umma_tf32_ss(tmem + h * 256, ad, bd, idesc, (kb | k) != 0);
        }
      }
      umma_commit(&empty[s]);
    }
    umma_commit(&tfull);
  }
  __syncwarp();
  // ---------------- epilogue: all 4 warps, warp w owns TMEM lanes 32w..32w+31 (= images of each batch tile)
  mbar_wait(&tfull, 0);
  tc_fence_after();
  const bool vec_ok = (N % 8) == 0;
  for (int hc = 0; hc < MB * BN; hc += 32) {
    const int h = hc / BN, c = hc % BN;
    const int b = b0 + h * PX_BM + warp * 32 + lane;
    const bool row_ok = b < batch;
    uint32_t r[32];
    tmem_ld32(tmem + h * 256 + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_ld_wait();
    const int col = n0 + c;
    if (!row_ok || col >= N) continue;
    if (ELT == 2 && !OF32) {
      __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(xt) + (size_t)b * N + col;
      if (vec_ok && col + 32 <= N) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 v;
          v.x = pack_bf16x2(__uint_as_float(r[8 * q + 0]), __uint_as_float(r[8 * q + 1]));
          v.y = pack_bf16x2(__uint_as_float(r[8 * q + 2]), __uint_as_float(r[8 * q + 3]));
          v.z = pack_bf16x2(__uint_as_float(r[8 * q + 4]), __uint_as_float(r[8 * q + 5]));
          v.w = pack_bf16x2(__uint_as_float(r[8 * q + 6]), __uint_as_float(r[8 * q + 7]));
          reinterpret_cast<uint4*>(dst)[q] = v;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (col + j < N) dst[j] = __float2bfloat16_rn(__uint_as_float(r[j]));
      }
    } else {
      float* dst;
      if (sc.world > 0) {   // row-sharded Phi: straight into the owner's slot for this rank (peer memory)
        const int r = b / sc.nb;
        dst = sc.slots[r] + ((size_t)sc.rank * sc.nb + (b - r * sc.nb)) * N + col;
      } else {
        dst = reinterpret_cast<float*>(xt) + (size_t)b * N + col;
      }
      if ((N % 4) == 0 && col + 32 <= N) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          reinterpret_cast<float4*>(dst)[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                                          __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (col + j < N) dst[j] = __uint_as_float(r[j]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<256 * MB>(tmem);
}

// ============================================================================ lifting GEMM on CTA pairs (cta_group::2)
// Large Phi (Stress: 2.15 GB, streamed from HBM once): a CTA pair computes a 256-image x 2 BN-pixel tile with
// M = 256 UMMAs (cta_group::2): each CTA stages ITS 128 images of Y (16 KB per K-block) and HALF of each of the two
// BN-row Phi^T blocks (BN / 2 rows each), the leader issues D[256][BN] += A[256][64] B[BN][64]^T for both pixel blocks
// (two TMEM accumulators, 2 x 256 columns in each CTA: rows 0..127 in the leader, 128..255 in the peer).  Per K-block
// an SM ingests 16 KB + BN x 128 B for 2 x 4 M=128-equivalent MMAs of N = BN, against 32 KB + BN x 128 B for the same
// MMA time with one CTA owning both batch tiles (k_proxy_tc MB = 2): the Y traffic per SM halves.
// Pipeline: full[s] lives in the leader (expect_tx of both CTAs' bytes, armed by the leader's producer; the peer's
// loads complete on it through the cluster window), empty[s] / tfull in both CTAs (multicast commits).
template <int BN>
__global__ void __launch_bounds__(128, 1)
    k_proxy_pair(const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmPh, int batch, int N,
                 int kblocks, __nv_bfloat16* __restrict__ xt) {
  constexpr uint32_t A_BYTES = 128 * 128, BH_BYTES = (BN / 2) * 128;   // per CTA: 128 images; BN/2 rows per block
  constexpr uint32_t STAGE = A_BYTES + 2 * BH_BYTES;
  constexpr int NST = PX2_STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ uint64_t full[NST], empty[NST], tfull;
  __shared__ uint32_t tslot;
  const int warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const int nbt = (batch + 255) / 256;
  const int bt = pair % nbt, pt = pair / nbt;            // consecutive pairs share one Phi^T slice (L2)
  const int b0 = bt * 256 + (int)rank * 128;             // this CTA's 128 images
  const int blk0 = 2 * pt;                               // the pair's two BN-pixel Phi^T blocks

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmY);
    tma_prefetch_desc(&tmPh);
    for (int s = 0; s < NST; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    mbar_init(&tfull, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair<512>(&tslot), tmem_relinquish_pair();
  tc_fence_before();
  cluster_sync_all();   // both CTAs' barriers initialised and TMEM allocated before any remote arrive / MMA
  tc_fence_after();
  const uint32_t tmem = tslot;
  griddep_wait();                 // the preceding grid's outputs (PDL: only the prologue above overlapped it)
  griddep_launch_dependents();

  if (warp == 0 && lane == 0) {  // ---------------- TMA producer (both CTAs)
    const int nblk = (N + BN - 1) / BN;
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % NST;
      if (kb >= NST) mbar_wait(&empty[s], ((kb / NST) - 1) & 1);
      uint8_t* sa = smem + s * STAGE;
      const uint32_t fbar = mapa_shared(&full[s], 0);
      if (rank == 0) mbar_arrive_expect_tx_cluster(fbar, 2 * STAGE);
      tma_load_2d_pair(sa, &tmY, fbar, kb * 64, b0);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int blk = min(blk0 + h, nblk - 1);   // a missing second block re-reads the first (outputs discarded)
        tma_load_3d_pair(sa + A_BYTES + h * BH_BYTES, &tmPh, fbar, 0, (int)rank * (BN / 2), blk * kblocks + kb);
      }
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {  // ---------------- MMA issuer (leader)
    constexpr uint32_t idesc = idesc_f32acc(1, 256, BN);
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % NST;
      mbar_wait(&full[s], (kb / NST) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * STAGE);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t ad = smem_desc(sa + k * 32, 16, 1024, kSwizzle128B);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint64_t bd = smem_desc(sa + A_BYTES + h * BH_BYTES + k * 32, 16, 1024, kSwizzle128B);
          umma_f16_ss_pair(tmem + h * 256, ad, bd, idesc, (kb | k) != 0);
        }
      }
      umma_commit_pair(&empty[s], 0x3);
    }
    umma_commit_pair(&tfull, 0x3);
  }
  __syncwarp();
  // ---------------- epilogue: each CTA's 4 warps, warp w = TMEM lanes 32w.. = images b0 + 32w + lane
  mbar_wait(&tfull, 0);
  tc_fence_after();
  const int b = b0 + warp * 32 + lane;
  const bool vec_ok = (N % 8) == 0;
  for (int hc = 0; hc < 2 * BN; hc += 32) {
    const int h = hc / BN, c = hc % BN;
    uint32_t r[32];
    tmem_ld32(tmem + h * 256 + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_ld_wait();
    const int col = (blk0 + h) * BN + c;
    if (b >= batch || col >= N) continue;
    __nv_bfloat16* dst = xt + (size_t)b * N + col;
    if (vec_ok && col + 32 <= N) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 v;
        v.x = pack_bf16x2(__uint_as_float(r[8 * q + 0]), __uint_as_float(r[8 * q + 1]));
        v.y = pack_bf16x2(__uint_as_float(r[8 * q + 2]), __uint_as_float(r[8 * q + 3]));
        v.z = pack_bf16x2(__uint_as_float(r[8 * q + 4]), __uint_as_float(r[8 * q + 5]));
        v.w = pack_bf16x2(__uint_as_float(r[8 * q + 6]), __uint_as_float(r[8 * q + 7]));
        reinterpret_cast<uint4*>(dst)[q] = v;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col + j < N) dst[j] = __float2bfloat16_rn(__uint_as_float(r[j]));
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();   // the peer's epilogue is done with its TMEM columns too
  if (warp == 2) tmem_dealloc_pair<512>(tmem);
}

template <int BN>
static size_t px2_smem() { return (size_t)PX2_STAGES * (128 * 128 + BN * 128) + 1024; }

cudaError_t setup_proxy_pair() {
  cudaError_t e = cudaFuncSetAttribute(k_proxy_pair<224>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)px2_smem<224>());
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_proxy_pair<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)px2_smem<256>());
}

// tmPh: tile-blocked Phi^T with a box of BN / 2 rows (encode_phiT_blk(..., half = true)); bn = the block width
cudaError_t launch_proxy_pair(const CUtensorMap* tmY, const CUtensorMap* tmPh, int batch, int N, int kblocks, void* xt,
                              int bn, cudaStream_t st) {
  const int nbt = (batch + 255) / 256, npt = (N + 2 * bn - 1) / (2 * bn);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * nbt * npt), cfg.blockDim = dim3(128), cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2, at[0].val.clusterDim.y = 1, at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL: the kernel waits in griddep_wait
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at, cfg.numAttrs = 2;
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(xt);
  if (bn == 224) {
    cfg.dynamicSmemBytes = px2_smem<224>();
    return cudaLaunchKernelEx(&cfg, k_proxy_pair<224>, *tmY, *tmPh, batch, N, kblocks, out);
  }
  if (bn != 256) return cudaErrorInvalidValue;
  cfg.dynamicSmemBytes = px2_smem<256>();
  return cudaLaunchKernelEx(&cfg, k_proxy_pair<256>, *tmY, *tmPh, batch, N, kblocks, out);
}

size_t proxy_tc_smem_bytes() { return (size_t)PX_STAGES * (PX_BM + PX_BN) * 128 + 1024; }
template <int MB, int BN>
static size_t px_smem() { return (size_t)(MB == 1 ? PX_STAGES : 3) * (MB * PX_BM + BN) * 128 + 1024; }

template <int ELT, bool OF32, int MB, int BN>
static void px_launch(const CUtensorMap* tmY, const CUtensorMap* tmPt, int batch, int N, int kblocks, void* xt,
                      cudaStream_t st, const ProxyScatter& s0, int bb) {
  const int nbt = (batch + PX_BM * MB - 1) / (PX_BM * MB), nnt = (N + BN - 1) / BN;
  launch_ex(k_proxy_tc<ELT, OF32, MB, BN>, dim3(nbt * nnt), dim3(128), px_smem<MB, BN>(), st, 1, true, *tmY, *tmPt, batch,
            N, kblocks, xt, s0, bb);
}
template <int ELT, bool OF32, int MB, int BN>
static cudaError_t px_setup() {
  return cudaFuncSetAttribute(k_proxy_tc<ELT, OF32, MB, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)px_smem<MB, BN>());
}

int proxy_tile_width(long long N, int max_batch, bool bf16, int num_sms) {
  if (!bf16) return PX_BN;
  const long long nbt = (max_batch + PX_BM - 1) / PX_BM, per = nbt % 2 == 0 ? nbt / 2 : nbt;
  double best = 0.0;
  int pick = PX_BN;
  for (int bn : {PX_BN, 224}) {   // fraction of the issued tile slots that hold real pixels
    const long long nnt = (N + bn - 1) / bn, ctas = per * nnt, waves = (ctas + num_sms - 1) / num_sms;
    const double eff = (double)ctas / (double)(waves * num_sms) * (double)N / (double)(nnt * bn);
    if (eff > best + 1e-9) best = eff, pick = bn;
  }
  return pick;
}

cudaError_t launch_proxy_tc(const CUtensorMap* tmY, const CUtensorMap* tmPt, int batch, int N, int kblocks,
                            void* xt, bool tf32, cudaStream_t st, bool out_f32, const ProxyScatter* sc, bool b_blocked,
                            int bn) {
  const int bb = b_blocked ? 1 : 0;
  const int nbt = (batch + PX_BM - 1) / PX_BM;
  ProxyScatter s0{};
  if (sc) s0 = *sc;
  const bool of = out_f32 || sc != nullptr;
  if (tf32) {
    if (bn != PX_BN) return cudaErrorInvalidValue;
    px_launch<4, true, 1, PX_BN>(tmY, tmPt, batch, N, kblocks, xt, st, s0, bb);
  } else if (nbt % 2 == 0) {   // pairs of batch tiles share each Phi^T K-block
    if (bn == 224)
      of ? px_launch<2, true, 2, 224>(tmY, tmPt, batch, N, kblocks, xt, st, s0, bb)
         : px_launch<2, false, 2, 224>(tmY, tmPt, batch, N, kblocks, xt, st, s0, bb);
    else
      of ? px_launch<2, true, 2, PX_BN>(tmY, tmPt, batch, N, kblocks, xt, st, s0, bb)
         : px_launch<2, false, 2, PX_BN>(tmY, tmPt, batch, N, kblocks, xt, st, s0, bb);
  } else {
    if (bn == 224)
      of ? px_launch<2, true, 1, 224>(tmY, tmPt, batch, N, kblocks, xt, st, s0, bb)
         : px_launch<2, false, 1, 224>(tmY, tmPt, batch, N, kblocks, xt, st, s0, bb);
    else
      of ? px_launch<2, true, 1, PX_BN>(tmY, tmPt, batch, N, kblocks, xt, st, s0, bb)
         : px_launch<2, false, 1, PX_BN>(tmY, tmPt, batch, N, kblocks, xt, st, s0, bb);
  }
  return cudaGetLastError();
}

cudaError_t setup_proxy_tc() {
  cudaError_t e;
  if ((e = px_setup<2, false, 1, PX_BN>()) != cudaSuccess) return e;
  if ((e = px_setup<2, true, 1, PX_BN>()) != cudaSuccess) return e;
  if ((e = px_setup<2, false, 2, PX_BN>()) != cudaSuccess) return e;
  if ((e = px_setup<2, true, 2, PX_BN>()) != cudaSuccess) return e;
  if ((e = px_setup<2, false, 1, 224>()) != cudaSuccess) return e;
  if ((e = px_setup<2, true, 1, 224>()) != cudaSuccess) return e;
  if ((e = px_setup<2, false, 2, 224>()) != cudaSuccess) return e;
  if ((e = px_setup<2, true, 2, 224>()) != cudaSuccess) return e;
  return px_setup<4, true, 1, PX_BN>();
}

// FP32 contexts: rows of a local partial to the owners' slots
__global__ void k_scatter_rows(const float* __restrict__ src, int batch, int N, ProxyScatter sc) {
  const size_t total = (size_t)batch * N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int b = (int)(i / N), j = (int)(i - (size_t)b * N), r = b / sc.nb;
    sc.slots[r][((size_t)sc.rank * sc.nb + (b - r * sc.nb)) * N + j] = src[i];
  }
}

cudaError_t launch_scatter_rows(const float* src, int batch, int N, const ProxyScatter* sc, cudaStream_t st) {
  k_scatter_rows<<<4 * 148, 256, 0, st>>>(src, batch, N, *sc);
  return cudaGetLastError();
}

// the owner's reduction: x_tilde[b][j] = sum_{r = 0..world-1} staging[r][b][j], in rank order (deterministic)
__global__ void k_reduce_slots(const float* __restrict__ staging, int world, int nb, int N, void* __restrict__ out,
                               int bf16) {
  const size_t total = (size_t)nb * N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int r = 0; r < world; ++r) acc += staging[(size_t)r * total + i];
    if (bf16)
      reinterpret_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(acc);
    else
      reinterpret_cast<float*>(out)[i] = acc;
  }
}

cudaError_t launch_reduce_slots(const float* staging, int world, int nb, int N, void* out, bool bf16, cudaStream_t st) {
  k_reduce_slots<<<4 * 148, 256, 0, st>>>(staging, world, nb, N, out, bf16 ? 1 : 0);
  return cudaGetLastError();
}

// fp32 -> bf16 (RNE), any n: a summed row-sharded proxy rounded once to the bf16 path's x_tilde
__global__ void k_round_bf16(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16_rn(src[i]);
}

cudaError_t launch_round_bf16(const float* src, void* dst, size_t n, cudaStream_t st) {
  k_round_bf16<<<4 * 148, 256, 0, st>>>(src, reinterpret_cast<__nv_bfloat16*>(dst), n);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- fp32 SIMT GEMM
// xt[b][j] = sum_i y[b][i] * phi[i][j];  64 (b) x 64 (j) tile, 256 threads, 4x4 outputs each.
__global__ void __launch_bounds__(256) k_proxy_f32(const float* __restrict__ y, long long ldy,
                                                   const float* __restrict__ phi, int m, int N, int batch,
                                                   float* __restrict__ xt) {
  __shared__ float sy[16][64 + 4];
  __shared__ float sp[16][64];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int j0 = blockIdx.x * 64, b0 = blockIdx.y * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < m; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int kk = e / 64, c = e % 64;
      const int bb = b0 + c, k = k0 + kk, jj = j0 + c;
      sy[kk][c] = (bb < batch && k < m) ? y[(size_t)bb * ldy + k] : 0.f;
      sp[kk][c] = (k < m && jj < N) ? phi[(size_t)k * N + jj] : 0.f;
    }
    __syncthreads();
    float part[4][4] = {};
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sy[kk][ty * 4 + i], bv[i] = sp[kk][tx + 16 * i];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) part[i][q] = fmaf(a[i], bv[q], part[i][q]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[i][q] += part[i][q];
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int bb = b0 + ty * 4 + i;
    if (bb >= batch) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int jj = j0 + tx + 16 * q;
      if (jj < N) xt[(size_t)bb * N + jj] = acc[i][q];
    }
  }
}

cudaError_t launch_proxy_f32(const float* y, long long ldy, const float* phi, int m, int N, int batch, float* xt,
                             cudaStream_t st) {
  dim3 grid((N + 63) / 64, (batch + 63) / 64);
  k_proxy_f32<<<grid, 256, 0, st>>>(y, ldy, phi, m, N, batch, xt);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- packing helpers
// Phi [m][N] (fp32 on device) -> Phi^T [N][kpad] in storage type (bf16 RNE or fp32), zero K tail.
template <typename T>
__global__ void k_pack_phiT(const float* __restrict__ phi, int m, int N, int kpad, int tr, T* __restrict__ out) {
  __shared__ float tile[32][33];
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int i = i0 + r, j = j0 + threadIdx.x;
    tile[r][threadIdx.x] = (i < m && j < N) ? phi[(size_t)i * N + j] : 0.f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int j = j0 + r, i = i0 + threadIdx.x;
    if (j < N && i < kpad) {
      const float v = tile[threadIdx.x][r];
      const size_t o = phiT_blk_index(j, i, kpad, 128 / (int)sizeof(T), tr);
      if constexpr (sizeof(T) == 2)
        out[o] = __float2bfloat16_rn(v);
      else
        out[o] = v;
    }
  }
}

cudaError_t launch_pack_phiT(const float* phi, int m, int N, int kpad, int tr, void* out, bool bf16, cudaStream_t st) {
  dim3 grid((N + 31) / 32, (kpad + 31) / 32), block(32, 8);
  if (bf16)
    k_pack_phiT<__nv_bfloat16><<<grid, block, 0, st>>>(phi, m, N, kpad, tr, reinterpret_cast<__nv_bfloat16*>(out));
  else
    k_pack_phiT<float><<<grid, block, 0, st>>>(phi, m, N, kpad, tr, reinterpret_cast<float*>(out));
  return cudaGetLastError();
}

// y [batch][ldy] (any alignment) -> packed [batch][kpad] with zero tail, same element type
template <typename T>
__global__ void k_stage_y(const T* __restrict__ y, long long ldy, int m, int kpad, int batch, T* __restrict__ out) {
  const long long total = (long long)batch * kpad;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / kpad;
    const int k = (int)(e - b * kpad);
    out[e] = k < m ? y[b * ldy + k] : T(0.f);
  }
}

cudaError_t launch_stage_y(const void* y, long long ldy, int m, int kpad, int batch, void* out, bool bf16,
                           cudaStream_t st) {
  const long long total = (long long)batch * kpad;
  const int blocks = (int)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
  if (bf16)
    k_stage_y<__nv_bfloat16><<<blocks, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(y), ldy, m, kpad,
                                                     batch, reinterpret_cast<__nv_bfloat16*>(out));
  else
    k_stage_y<float><<<blocks, 256, 0, st>>>(reinterpret_cast<const float*>(y), ldy, m, kpad, batch,
                                            reinterpret_cast<float*>(out));
  return cudaGetLastError();
}

DI_DEBUG_BINDER(di_debug_bind_k_proxy)

}  // namespace di
