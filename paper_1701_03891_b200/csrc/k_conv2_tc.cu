// k_conv2_tc.cu -- stage 2, conv layer 2 of DeepInverse (32 filters 11x11x64 + bias + ReLU, crop S;
// PAPER.md:130-131, 150; Eq. (1)) on the 5th-generation tensor cores.  ~90 % of the
// path's FLOPs.
//
// Formulation: 'same' cross-correlation with the flipped taps W'
//   h2[k][r][c] = ReLU( sum_{ci,a,b} W'[k][ci][a][b] * h1[ci][r+a-5][c+b-5] + bias )
// as an implicit GEMM with PIXELS IN THE UMMA N DIMENSION and four column taps stacked in M:
//   A (M=128 rows = 4 taps v' x 32 filters k, K = 64 input channels) = packed weights of K-block (u, v0),
//   B (N <= 256 rows = consecutive positions of a zero-padded strip, K = 64 channels) = a window of the
//     shared-memory activation strip starting at position n0 + u*P + v0 (a plain 128-B-row offset of the
//     SWIZZLE_128B tile; verified on B200: the UMMA swizzle is address-based, base_offset = 0),
//   D[v'*32 + k][n] accumulates over the 33 K-blocks (u = 0..10, v0 = 0,4,8; tap v0+v' = 11 is zero),
//   so output position o = n0 + j receives  sum_v' D[v'*32+k][j + v'].
// The epilogue reads each tap group v' from its own TMEM lane quadrant at a column offset of v'
// (one tcgen05.ld per warp), sums the 4 quadrants through shared memory, adds the bias, applies
// ReLU, rounds to bf16 and stores NHWC h2 with 16-B coalesced stores.
//
// Work unit = (image b, 6 output rows from r0, <=64 output columns from c0).  The strip of the unit
// ((6+10) rows x (W+10) columns x 64 ch, bf16) is loaded by ONE 4-D TMA box whose out-of-bounds
// elements are zero: that is the zero padding of Eq. (1) at the image border.
// Positions are linear in the padded strip (pitch P = W+10); tiles of 256 positions overlap by 3.
//
// Roles (256 threads): warp 0 TMA producer (strip + 16-KB weight K-blocks via bulk copies, 3 stages),
// warp 1 single-thread MMA issuer, warp 2 TMEM allocator, warps 4..7 epilogue (one TMEM lane quadrant each).
// TMEM: two 256-column fp32 accumulators (double buffer: MMA of tile i+1 overlaps the epilogue of tile i).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "sm100.cuh"

namespace di {

namespace {
constexpr int R = C2_ROWS;             // output rows per unit (6)
constexpr int WSEG = 64;               // output columns per unit (max)
constexpr int NT = 256;                // UMMA N per tile
constexpr int OUT_PER_TILE = NT - 3;   // 253 complete output positions per tile
constexpr int WSTAGES = 3;
constexpr int KBLOCKS = C2_KBLOCKS;    // 33
constexpr uint32_t WBYTES = C2_KBLOCK_BYTES;  // 16 KB
constexpr int GUARD_ROWS = 24;

struct Geo {
  int n1, n2, wseg, P, nrb, ncs, units;
};

__host__ __device__ inline int strip_rows_bytes(int P) { return (R + 10) * P * 128; }
}  // namespace

// last chunk of a full tile (c0 = 224, at most 29 outputs): columns c0+q .. c0+q+28 <= 255, loaded as
// 16 + 8 + 4 + 1 columns at fixed register offsets (no dynamic register indexing)
__device__ __forceinline__ void ld_tail29(uint32_t taddr, uint32_t* r) {
  tmem_ld16(taddr, r);
  tmem_ld8(taddr + 16, r + 16);
  tmem_ld4(taddr + 24, r + 24);
  tmem_ld1(taddr + 28, r + 28);
}

__global__ void __launch_bounds__(256, 1)
    k_conv2_tc(const __grid_constant__ CUtensorMap tmH1, const __nv_bfloat16* __restrict__ wpack,
               const float* __restrict__ bias, int fullmap, Geo g, __nv_bfloat16* __restrict__ h2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int strip_bytes = strip_rows_bytes(g.P);
  const int strip_alloc = (strip_bytes + GUARD_ROWS * 128 + 1023) & ~1023;
  uint8_t* strip = smem;
  uint8_t* wst = smem + strip_alloc;
  float* sP = reinterpret_cast<float*>(wst + WSTAGES * WBYTES);  // [4][32][32]

  __shared__ uint64_t strip_full, strip_empty, wfull[WSTAGES], wempty[WSTAGES], tfull[2], tempty[2];
  __shared__ uint32_t tslot;
  const int warp = warp_id(), lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmH1);
    mbar_init(&strip_full, 1);
    mbar_init(&strip_empty, 1);
    for (int s = 0; s < WSTAGES; ++s) mbar_init(&wfull[s], 1), mbar_init(&wempty[s], 1);
    for (int s = 0; s < 2; ++s) mbar_init(&tfull[s], 1), mbar_init(&tempty[s], 4);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&tslot), tmem_relinquish();
  // Guard rows after the strip: the zero tap slot (v = 11) of the last output position and the padded
  // columns of the last tile read up to GUARD_ROWS rows past the TMA box.  Their weights / outputs are
  // zero / discarded, but 0 * (NaN garbage) would not be, so the guard must hold finite values.
  for (int i = threadIdx.x; i < GUARD_ROWS * 128 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(strip + strip_bytes)[i] = make_uint4(0, 0, 0, 0);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;

  const int per_img = g.nrb * g.ncs;
  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ producer
      int wk = 0, it = 0;
      for (int u = blockIdx.x; u < g.units; u += gridDim.x, ++it) {
        const int b = u / per_img, rem = u - b * per_img;
        const int r0 = (rem / g.ncs) * R, c0 = (rem % g.ncs) * g.wseg;
        const int rows = min(R, g.n1 - r0);
        const int L = (rows - 1) * g.P + g.wseg;
        const int ntiles = (L + OUT_PER_TILE - 1) / OUT_PER_TILE;
        if (it > 0) mbar_wait(&strip_empty, (it - 1) & 1);
        mbar_arrive_expect_tx(&strip_full, strip_bytes);
        tma_load_4d(strip, &tmH1, &strip_full, 0, c0 - 5, r0 - 5, b);
        for (int t = 0; t < ntiles; ++t) {
          for (int kb = 0; kb < KBLOCKS; ++kb, ++wk) {
            const int s = wk % WSTAGES;
            if (wk >= WSTAGES) mbar_wait(&wempty[s], ((wk / WSTAGES) - 1) & 1);
            mbar_arrive_expect_tx(&wfull[s], WBYTES);
            bulk_load(wst + s * WBYTES, reinterpret_cast<const uint8_t*>(wpack) + (size_t)kb * WBYTES, WBYTES,
                      &wfull[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      int wk = 0, it = 0, ti = 0;
      const uint32_t strip_s = smem_u32(strip), wst_s = smem_u32(wst);
      for (int u = blockIdx.x; u < g.units; u += gridDim.x, ++it) {
        const int b = u / per_img, rem = u - b * per_img;
        const int r0 = (rem / g.ncs) * R;
        (void)b;
        const int rows = min(R, g.n1 - r0);
        const int L = (rows - 1) * g.P + g.wseg;
        const int ntiles = (L + OUT_PER_TILE - 1) / OUT_PER_TILE;
        mbar_wait(&strip_full, it & 1);
        tc_fence_after();
        for (int t = 0; t < ntiles; ++t, ++ti) {
          const int n0 = t * OUT_PER_TILE;
          const int cnt = min(OUT_PER_TILE, L - n0);
          const int nmma = min(NT, (cnt + 3 + 15) & ~15);
          const uint32_t idesc = idesc_f32acc(1, 128, nmma);
          const int buf = ti & 1;
          if (ti >= 2) mbar_wait(&tempty[buf], ((ti >> 1) - 1) & 1);
          tc_fence_after();
          const uint32_t d = tmem + buf * 256;
          for (int kb = 0; kb < KBLOCKS; ++kb, ++wk) {
            const int s = wk % WSTAGES;
            mbar_wait(&wfull[s], (wk / WSTAGES) & 1);
            tc_fence_after();
            const int uu = kb / 3, v0 = (kb - uu * 3) * 4;
            const uint32_t bpos = strip_s + (uint32_t)(n0 + uu * g.P + v0) * 128;
            const uint32_t apos = wst_s + s * WBYTES;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              umma_f16_ss(d, smem_desc(apos + k * 32, 16, 1024, kSwizzle128B),
                          smem_desc(bpos + k * 32, 16, 1024, kSwizzle128B), idesc, (kb | k) != 0);
            }
            umma_commit(&wempty[s]);
          }
          umma_commit(&tfull[buf]);
        }
        umma_commit(&strip_empty);
      }
    }
  } else if (warp >= 4) {  // ---------------------------------------------- epilogue
    const int q = warp - 4;              // TMEM lane quadrant = column-tap group v'
    const int e = threadIdx.x - 128;     // 0..127
    const int jj = e >> 2, kg = e & 3;   // reduce role: output position jj of the chunk, channels 8kg..8kg+7
    float bch[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) bch[i] = (!fullmap && bias) ? bias[8 * kg + i] : 0.f;
    int ti = 0;
    for (int u = blockIdx.x; u < g.units; u += gridDim.x) {
      const int b = u / per_img, rem = u - b * per_img;
      const int r0 = (rem / g.ncs) * R, c0 = (rem % g.ncs) * g.wseg;
      const int rows = min(R, g.n1 - r0);
      const int L = (rows - 1) * g.P + g.wseg;
      const int ntiles = (L + OUT_PER_TILE - 1) / OUT_PER_TILE;
      for (int t = 0; t < ntiles; ++t, ++ti) {
        const int n0 = t * OUT_PER_TILE;
        const int cnt = min(OUT_PER_TILE, L - n0);
        const int buf = ti & 1;
        mbar_wait(&tfull[buf], (ti >> 1) & 1);
        tc_fence_after();
        const uint32_t tq = tmem + buf * 256 + ((uint32_t)(q * 32) << 16);
        for (int c = 0; c < cnt; c += 32) {
          const int nout = min(32, cnt - c);
          uint32_t r[32];
          if (c + q + 32 <= NT)
            tmem_ld32(tq + c + q, r);
          else
            ld_tail29(tq + c + q, r);
          tmem_ld_wait();
          float* dst = sP + q * 1024 + lane;   // sP[q][j][k], k = lane
#pragma unroll
          for (int j = 0; j < 32; ++j) dst[j * 32] = __uint_as_float(r[j]);
          named_bar(1, 128);
          if (jj < nout) {
            const int o = n0 + c + jj;
            const int rr = o / g.P, cc = o - rr * g.P;
            const int orow = r0 + rr, ocol = c0 + cc;
            if (cc < g.wseg && ocol < g.n2 && orow < g.n1) {
              float s[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) s[i] = 0.f;
#pragma unroll
              for (int qq = 0; qq < 4; ++qq) {
                const float4* p = reinterpret_cast<const float4*>(sP + qq * 1024 + jj * 32 + 8 * kg);
                const float4 a = p[0], bq = p[1];
                s[0] += a.x, s[1] += a.y, s[2] += a.z, s[3] += a.w;
                s[4] += bq.x, s[5] += bq.y, s[6] += bq.z, s[7] += bq.w;
              }
              const size_t pix = ((size_t)b * g.n1 + orow) * g.n2 + ocol;
              if (fullmap && bias) {
                const float4* bp = reinterpret_cast<const float4*>(bias + pix % ((size_t)g.n1 * g.n2) * 32 + 8 * kg);
                const float4 a = bp[0], bq = bp[1];
                s[0] += a.x, s[1] += a.y, s[2] += a.z, s[3] += a.w;
                s[4] += bq.x, s[5] += bq.y, s[6] += bq.z, s[7] += bq.w;
              } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) s[i] += bch[i];
              }
              uint4 v;
              v.x = pack_bf16x2(fmaxf(s[0], 0.f), fmaxf(s[1], 0.f));
              v.y = pack_bf16x2(fmaxf(s[2], 0.f), fmaxf(s[3], 0.f));
              v.z = pack_bf16x2(fmaxf(s[4], 0.f), fmaxf(s[5], 0.f));
              v.w = pack_bf16x2(fmaxf(s[6], 0.f), fmaxf(s[7], 0.f));
              *reinterpret_cast<uint4*>(h2 + pix * 32 + 8 * kg) = v;
            }
          }
          named_bar(1, 128);
        }
        tc_fence_before();
        if (lane == 0) mbar_arrive(&tempty[buf]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

static Geo make_geo(int batch, int n1, int n2) {
  Geo g;
  g.n1 = n1, g.n2 = n2;
  g.wseg = n2 < WSEG ? n2 : WSEG;
  g.P = g.wseg + 10;
  g.nrb = (n1 + R - 1) / R;
  g.ncs = (n2 + g.wseg - 1) / g.wseg;
  g.units = batch * g.nrb * g.ncs;
  return g;
}

size_t conv2_tc_smem_bytes(int n2) {
  const int wseg = n2 < WSEG ? n2 : WSEG, P = wseg + 10;
  const size_t strip_alloc = ((size_t)strip_rows_bytes(P) + GUARD_ROWS * 128 + 1023) & ~(size_t)1023;
  return strip_alloc + WSTAGES * WBYTES + 4 * 32 * 32 * 4 + 1024;
}

int conv2_tc_box_rows() { return R + 10; }
int conv2_tc_box_cols(int n2) { return (n2 < WSEG ? n2 : WSEG) + 10; }

cudaError_t setup_conv2_tc(int n2) {
  return cudaFuncSetAttribute(k_conv2_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)conv2_tc_smem_bytes(n2));
}

cudaError_t launch_conv2_tc(const CUtensorMap* tmH1, const void* wpack, const float* bias, int fullmap, int batch,
                            int n1, int n2, void* h2, int num_sms, cudaStream_t st) {
  Geo g = make_geo(batch, n1, n2);
  const int grid = g.units < num_sms ? g.units : num_sms;
  k_conv2_tc<<<grid, 256, conv2_tc_smem_bytes(n2), st>>>(*tmH1, reinterpret_cast<const __nv_bfloat16*>(wpack), bias,
                                                         fullmap, g, reinterpret_cast<__nv_bfloat16*>(h2));
  return cudaGetLastError();
}

}  // namespace di
