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
// Work unit = (image b, R = 6 output rows from r0, <=64 output columns from c0).  The strip of the unit
// ((R+10) rows x (W+10) columns x 64 ch, bf16) is loaded by ONE 4-D TMA box whose out-of-bounds
// elements are zero: that is the zero padding of Eq. (1) at the image border.
// Positions are linear in the padded strip (pitch P = W+5, or 74 for several column segments); tiles of 256
// positions overlap by 3.
//
// Roles (256 threads): warp 0 producer (strip by TMA at unit start, 16-KB weight K-blocks by bulk copies into a
// 4-deep ring), warp 1 single-thread MMA issuer (lean loop: prebuilt descriptors), warp 2 TMEM allocator,
// warps 4..7 epilogue (one TMEM lane quadrant each, conflict-free 16-position shared-memory transpose).
// TMEM: two 256-column fp32 accumulators (double buffer: MMA of tile i+1 overlaps the epilogue of tile i).
// Bound: the shared-memory port (A + B operand reads + weight fills ~ 121 B/clk of ~128), DESIGN.md §6.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "kernels.cuh"
#define DI_TU_ID 3
#include "sm100.cuh"

namespace di {

namespace {
constexpr int R = C2_ROWS;             // output rows per unit (6)
constexpr int WSEG = 64;               // output columns per unit (max)
constexpr int NT = 256;                // UMMA N per tile
constexpr int OUT_PER_TILE = NT - 3;   // 253 complete output positions per tile
#ifndef DI_C2_WSTAGES
#define DI_C2_WSTAGES 4
#endif
constexpr int WSTAGES = DI_C2_WSTAGES;  // weight ring depth (a 16-KB bulk copy takes ~1.4k cycles to land)
constexpr int KBLOCKS = C2_KBLOCKS;    // 33
constexpr uint32_t WBYTES = C2_KBLOCK_BYTES;  // 16 KB
constexpr int GUARD_ROWS = 24;
constexpr int SPS = 36;                  // epilogue transpose row stride (floats): conflict-free float4 reads
constexpr int ECH = 16;                  // epilogue chunk: output positions per TMEM load
constexpr int C2_WST64 = 12;             // weight stages of the 64-B-row instance (8 KB each)
// output rows per unit of the 64-B-row instance (the layer-2 dgrad): every tile restreams the 528 KB of packed weights,
// and that stream bounds the instance, so its units are taller -- 3 tiles of ~253 outputs per 11-row unit (18 tiles
// per 64-row image) instead of 2 of 253 + 156 per 6-row unit (22 tiles)
constexpr int C2_DG_ROWS = 11;

struct Geo {
  int n1, n2, wseg, P, nrb, ncs, units;
  int balanced;   // 1: a unit's tiles share its outputs evenly (2 x 205 at 64 x 64); 0: 253 + the rest
  int nfull;      // row blocks whose units have the full tile count; units of the others are enumerated last
  int batch;
  int ntall;      // the first ntall row blocks of an image are R + 1 rows tall (mixed heights, conv2_tc_tall_blocks)
  int srows;      // strip rows loaded per unit (the TMA box): R + 10, or R + 11 with tall blocks
};
// Unit u -> (image b, first output row r0, rows, first column c0).  Units of the nfull full-height row blocks of
// every image come first, then those of the remaining (shorter, fewer-tile) row blocks: the two CTAs of a
// weight-multicast pair (units u and u + 1 at every step of the grid stride) then always run the same number of
// tiles.  With mixed heights the nfull = ntall tall blocks come first, then the R-row ones (both two tiles).
__device__ __forceinline__ void unit_of(const Geo& g, int u, int R, int& b, int& r0, int& rows, int& c0) {
  const int nf = g.nfull * g.ncs, split = g.batch * nf;
  int rb, cs;
  if (u < split) {
    b = u / nf;
    const int rem = u - b * nf;
    rb = rem / g.ncs, cs = rem - (rem / g.ncs) * g.ncs;
  } else {
    const int v = u - split, ns = (g.nrb - g.nfull) * g.ncs;
    b = v / ns;
    const int rem = v - b * ns;
    rb = g.nfull + rem / g.ncs, cs = rem - (rem / g.ncs) * g.ncs;
  }
  r0 = rb * R + min(rb, g.ntall), c0 = cs * g.wseg;
  rows = min(R + (rb < g.ntall ? 1 : 0), g.n1 - r0);
}
// Tile t of a unit with L output positions: [n0, n0 + cnt).  Balanced tiles give every tile the same MMA length,
// so the weight stream (33 K-blocks per tile, whatever its width) is consumed at one even rate instead of a burst
// during the short second tile.  A tile of cnt outputs runs N = cnt + 3 rounded up to 16 MMA columns; when the even
// share rounds up (478 = 2 x 239 -> 2 x 256 columns), the first tiles take the largest span that fits one column
// step less (237 -> 240 columns, the last 241 -> 256) if the last tile still fits.
__host__ __device__ inline int tile_span(const Geo& g, int L, int& ntiles) {
  ntiles = (L + OUT_PER_TILE - 1) / OUT_PER_TILE;
  if (!g.balanced) return OUT_PER_TILE;
  const int s = (L + ntiles - 1) / ntiles, sf = ((s + 3) & ~15) - 3, lf = L - (ntiles - 1) * sf;
  auto cols = [&](int span, int last) { return (ntiles - 1) * ((span + 3 + 15) & ~15) + ((last + 3 + 15) & ~15); };
  return sf > 0 && lf <= OUT_PER_TILE && cols(sf, lf) < cols(s, L - (ntiles - 1) * s) ? sf : s;
}

__host__ __device__ inline int strip_rows_bytes(int rows, int P) { return rows * P * 128; }   // C_in = 64
}  // namespace

// last chunk of a full tile (c0 = 224, at most 29 outputs): columns c0+q .. c0+q+28 <= 255, loaded as
// 16 + 8 + 4 + 1 columns at fixed register offsets (no dynamic register indexing)
// last 16-column chunk of a full tile (c0 = 240, at most 13 outputs): columns c0+q .. c0+q+12 <= 255
__device__ __forceinline__ void ld_tail13(uint32_t taddr, uint32_t* r) {
  tmem_ld8(taddr, r);
  tmem_ld4(taddr + 8, r + 8);
  tmem_ld1(taddr + 12, r + 12);
}


enum { C2_BIAS_RELU = 0, C2_MASK = 1 };

// Template over the channel counts (the paper's layer 2 is <64, 32, C2_BIAS_RELU>): TAPS = 128 / C_out column taps
// x C_out filters in M, strip rows of C_in bf16 channels (128 B: SWIZZLE_128B; 64 B: SWIZZLE_64B), K-block = one
// strip row (C_in / 16 MMAs of K = 16), 11 ceil(11 / TAPS) K-blocks per tile.  <32, 64, C2_MASK> is the training
// step's layer-2 data gradient: dG2 (bf16) in, the rotated bank, out = [h1 > 0] * conv in bf16 (mask = bf16 h1).
// MC: CTA pairs (cluster of 2) share the weight stream -- each CTA copies half of every K-block to BOTH CTAs'
// rings (multicast) and each MMA commit frees the stage in both, halving the L2 -> SM weight traffic.  Needs the two
// CTAs of a pair to consume the same K-block sequence (equal tile counts: launch_conv2_tc checks).
template <int CIN, int COUT, int MODE, int CL = 1>
__global__ void __launch_bounds__(COUT >= 64 ? 384 : 256, 1)
    k_conv2_tc(const __grid_constant__ CUtensorMap tmH1, const __nv_bfloat16* __restrict__ wpack,
               const float* __restrict__ bias, int fullmap, Geo g, __nv_bfloat16* __restrict__ h2,
               const __nv_bfloat16* __restrict__ mask) {
  constexpr int TAPS = 128 / COUT, J = (11 + TAPS - 1) / TAPS, KB = 11 * J;
  // C_in = 128 (custom stacks, NEXT-3): two 64-channel halves, each its own strip load and 11 J K-blocks per tile,
  // accumulated into the same TMEM tile (a 128-channel strip would need 283 KB of shared memory)
  constexpr int NH = CIN > 64 ? CIN / 64 : 1, CINH = CIN / NH;
  constexpr int RB = CINH * 2, KMMA = RB / 32;
  constexpr uint32_t WB = 128 * RB;
  constexpr uint32_t SWZ = RB == 128 ? kSwizzle128B : kSwizzle64B;
  constexpr int QPT = COUT / 32, CPT = COUT / 8;
  // epilogue groups: C_out = 64 (twice the epilogue work per tile) runs two groups of 4 warps, one per TMEM buffer
  constexpr int EG = COUT >= 64 ? 2 : 1;
  // weight ring: 4 stages of 16 KB for 128-B rows; 12 stages of 8 KB for 64-B rows (the layer-2 dgrad)
  constexpr int WST = RB == 128 ? (COUT >= 64 ? 3 : WSTAGES) : C2_WST64;   // C_out >= 64: room for 2 epilogue groups
  constexpr int R = RB == 128 ? C2_ROWS : C2_DG_ROWS;   // output rows per unit
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const int strip_bytes = g.srows * g.P * RB;
  const int strip_alloc = (strip_bytes + GUARD_ROWS * RB + 1023) & ~1023;
  uint8_t* strip = smem;
  uint8_t* wst = smem + strip_alloc;
  float* sP = reinterpret_cast<float*>(wst + WST * WB);  // [4][ECH positions][SPS]

  __shared__ uint64_t hfull[2], hempty[2], wfull[WST], wempty[WST], tfull[2], tempty[2];
#ifdef DI_PROF_CONV2
  __shared__ long long t_issue[WST];   // producer: clock64 when the copy of the stage's K-block was issued
#endif
  __shared__ uint32_t tslot;
  const int warp = warp_id(), lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmH1);
    for (int h = 0; h < 2; ++h) mbar_init(&hfull[h], 1), mbar_init(&hempty[h], 1);
    for (int s = 0; s < WST; ++s) mbar_init(&wfull[s], 1), mbar_init(&wempty[s], CL);
    for (int s = 0; s < 2; ++s) mbar_init(&tfull[s], 1), mbar_init(&tempty[s], 4);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&tslot), tmem_relinquish();
  // Guard rows after the strip: the zero tap slot (v = 11) of the last output position and the padded
  // columns of the last tile read up to GUARD_ROWS rows past the TMA box.  Their weights / outputs are
  // zero / discarded, but 0 * (NaN garbage) would not be, so the guard must hold finite values.
  for (int i = threadIdx.x; i < GUARD_ROWS * RB / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(strip + strip_bytes)[i] = make_uint4(0, 0, 0, 0);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync_all();   // the peers' barriers are initialised before any multicast copy or commit
  tc_fence_after();
  const uint32_t tmem = tslot;
  griddep_wait();                 // the preceding grid's outputs (PDL: only the prologue above overlapped it)
  griddep_launch_dependents();
  const uint32_t crank = CL > 1 ? cluster_ctarank() : 0;
  constexpr uint16_t CMASK = (uint16_t)((1u << CL) - 1);

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ strip + weight producer
      uint32_t wk = 0;                    // weight K-blocks issued (stage wk % WST)
      int it = 0, sl = 0;                 // units, strip loads
      for (int u = blockIdx.x; u < g.units; u += gridDim.x, ++it) {
        int b, r0, rows, c0;
        unit_of(g, u, R, b, r0, rows, c0);
        const int L = (rows - 1) * g.P + g.wseg;
        int ntiles;
        tile_span(g, L, ntiles);
        for (int t = 0; t < ntiles; ++t)
         for (int h = 0; h < NH; ++h) {
          if (NH > 1 || t == 0) {   // the unit's strip (C_in = 128: channel half h, per tile)
            if (sl > 0) mbar_wait(&hempty[0], (sl - 1) & 1);
            mbar_arrive_expect_tx(&hfull[0], strip_bytes);
            tma_load_4d(strip, &tmH1, &hfull[0], CINH * h, c0 - 5, r0 - 5, b);
            ++sl;
          }
          const uint8_t* wsrc = reinterpret_cast<const uint8_t*>(wpack) + (size_t)h * KB * WB;
          for (int kb = 0; kb < KB; ++kb, ++wk, wsrc += WB) {
            const uint32_t st = wk % WST;
            if (wk >= WST) mbar_wait(&wempty[st], ((wk / WST) - 1) & 1);
#ifdef DI_PROF_CONV2
            t_issue[st] = clock64();
#endif
            mbar_arrive_expect_tx(&wfull[st], WB);
            if (CL > 1)   // this CTA's 1/CL of the K-block, to every CTA of the cluster
              bulk_load_mc(wst + st * WB + crank * (WB / CL), wsrc + crank * (WB / CL), WB / CL, &wfull[st], CMASK);
            else
              bulk_load(wst + st * WB, wsrc, WB, &wfull[st]);
          }
        }
      }
      if (CL > 1)   // every commit (local and the peers') into this CTA's ring has landed before the cluster exits
        for (uint32_t k = wk > (uint32_t)WST ? wk - WST : 0; k < wk; ++k) mbar_wait(&wempty[k % WST], (k / WST) & 1);
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      // Lean loop: descriptors built once, per-MMA addresses are immediate 64-bit adds of (bytes >> 4); the
      // stage index of K-block (uu, j) is j (33 K-blocks per tile, 3 stages).  A single issuing thread is
      // latency-bound, so every instruction here costs tensor-pipe time.
      const uint64_t bdesc0 = smem_desc(smem_u32(strip), 16, 8 * RB, SWZ);
      const uint64_t adesc0 = smem_desc(smem_u32(wst), 16, 8 * RB, SWZ);
      const uint64_t pstep = (uint64_t)g.P * (RB >> 4);    // one tap row = P positions x RB bytes, >> 4
      uint32_t wk = 0;
      int it = 0, ti = 0, sl = 0;
#ifdef DI_PROF_CONV2
      long long c_h = 0, c_t = 0, c_w = 0, c_w0 = 0, c_w1 = 0, c0_ = clock64(), c_lat = 0, c_latmax = 0;
#define PT0 long long _t0 = clock64();
#define PT1(acc) acc += clock64() - _t0;
#else
#define PT0
#define PT1(acc)
#endif
      for (int u = blockIdx.x; u < g.units; u += gridDim.x, ++it) {
        int b_, r0, rows, c0_;
        unit_of(g, u, R, b_, r0, rows, c0_);
        const int L = (rows - 1) * g.P + g.wseg;
        int ntiles;
        const int span = tile_span(g, L, ntiles);
        for (int t = 0; t < ntiles; ++t, ++ti) {
          const int n0 = t * span;
          const int cnt = t == ntiles - 1 ? L - n0 : span;   // the last tile takes the rest (tile_span's short first tiles)
          const int nmma = min(NT, (cnt + TAPS - 1 + 15) & ~15);
          const uint32_t idesc = idesc_f32acc(1, 128, nmma);
          const int buf = ti & 1;
          { PT0 if (ti >= 2) mbar_wait(&tempty[buf], ((ti >> 1) - 1) & 1); PT1(c_t) }
          tc_fence_after();
          const uint32_t d = tmem + buf * 256;
          // the last K-block's window (u = 10, v0 = TAPS (J - 1)) stays inside the strip and its guard rows
          DI_DEVICE_ASSERT(n0 + 10 * g.P + TAPS * (J - 1) + nmma <= g.srows * g.P + GUARD_ROWS, n0, nmma);
         for (int h = 0; h < NH; ++h) {
          if (NH > 1 || t == 0) {
            { PT0 mbar_wait(&hfull[0], sl & 1); PT1(c_h) }
            tc_fence_after();
          }
          uint64_t bd = bdesc0 + (uint64_t)(n0 * (RB >> 4));
          for (int uu = 0; uu < 11; ++uu, bd += pstep) {
#pragma unroll
            for (int j = 0; j < J; ++j, ++wk) {   // column-tap groups v0 = TAPS j (0, 4, 8 for C_out = 32)
              const uint32_t st = wk % WST;
#ifdef DI_PROF_CONV2
              { PT0 mbar_wait(&wfull[st], (wk / WST) & 1);
                if (t == 0 && uu < 3) { PT1(c_w0) } else if (t == 0) { PT1(c_w) } else { PT1(c_w1) }
                const long long lat = clock64() - *(volatile long long*)&t_issue[st];
                c_lat += lat; c_latmax = max(c_latmax, lat); }
#else
              mbar_wait(&wfull[st], (wk / WST) & 1);
#endif
              tc_fence_after();
              const uint64_t ad = adesc0 + (uint64_t)(st * (WB >> 4));
              const uint64_t b = bd + (uint64_t)(TAPS * j * (RB >> 4));   // v0 = TAPS j positions
              umma_f16_ss(d, ad, b, idesc, (h | uu | j) != 0);
#pragma unroll
              for (int kk = 1; kk < KMMA; ++kk) umma_f16_ss(d, ad + 2 * kk, b + 2 * kk, idesc, 1);
              if (CL > 1)
                umma_commit_mc(&wempty[st], CMASK);
              else
                umma_commit(&wempty[st]);
            }
          }
          if (NH > 1) {   // this half's strip is free for the next load
            umma_commit(&hempty[0]);
            ++sl;
          }
         }
          umma_commit(&tfull[buf]);
        }
        if (NH == 1) {
          umma_commit(&hempty[0]);
          ++sl;
        }
      }
#ifdef DI_PROF_CONV2
      if (blockIdx.x % 37 == 0)
        printf("conv2 cta %d: cycles %lld strip-wait %lld tmem-wait %lld weight-wait first9 %lld tile0-rest %lld "
               "later-tiles %lld units %d kblocks %u | issue->ready mean %lld max %lld\n", blockIdx.x, clock64() - c0_,
               c_h, c_t, c_w0, c_w, c_w1, it, wk, c_lat / (long long)wk, c_latmax);
#endif
    }
  } else if (warp >= 4) {  // ---------------------------------------------- epilogue
    const int q = warp & 3;              // TMEM lane quadrant: column tap q / QPT, channel block q % QPT
    const int grp = (warp - 4) >> 2;     // epilogue group: TMEM buffer grp when EG = 2
    const int shift = q / QPT;
    const int e = (threadIdx.x - 128) & 127;
    float* const sPg = sP + grp * (4 * ECH * SPS);
    const int jj = e >> 3, kg = e & 7;   // reduce role: output position jj of the chunk, channels CPT kg ..
    const int c0ch = CPT * kg, cblk = c0ch / 32, cl = c0ch % 32;
    float bch[CPT];
#pragma unroll
    for (int i = 0; i < CPT; ++i) bch[i] = (MODE == C2_BIAS_RELU && !fullmap && bias) ? bias[c0ch + i] : 0.f;
    int ti = 0;
    for (int u = blockIdx.x; u < g.units; u += gridDim.x) {
      int b, r0, rows, c0;
      unit_of(g, u, R, b, r0, rows, c0);
      const int L = (rows - 1) * g.P + g.wseg;
      int ntiles;
      const int span = tile_span(g, L, ntiles);
      for (int t = 0; t < ntiles; ++t, ++ti) {
        const int n0 = t * span;
        const int cnt = t == ntiles - 1 ? L - n0 : span;
        const int buf = ti & 1;
        if (EG == 2 && buf != grp) continue;
        mbar_wait(&tfull[buf], (ti >> 1) & 1);
        tc_fence_after();
        const uint32_t tq = tmem + buf * 256 + ((uint32_t)(q * 32) << 16);
        // this thread's output of chunk cb (reduce role): valid?, pixel index
        auto outpos = [&](int cb, size_t& pix) {
          const int o = n0 + cb + jj;
          const int rr = o / g.P, cc = o - rr * g.P;
          const int orow = r0 + rr, ocol = c0 + cc;
          pix = ((size_t)b * g.n1 + orow) * g.n2 + ocol;
          return jj < min(ECH, cnt - cb) && cc < g.wseg && ocol < g.n2 && rr < rows;
        };
        // ReLU' mask of the thread's output, loaded one chunk ahead (its global latency overlaps a whole chunk)
        uint2 mn[CPT / 4];
        auto mask_ld = [&](int cb) {
          size_t px;
          const bool v = outpos(cb, px);
#pragma unroll
          for (int v4 = 0; v4 < CPT / 4; ++v4)
            mn[v4] = v ? __ldg(reinterpret_cast<const uint2*>(mask + px * COUT + c0ch + 4 * v4)) : make_uint2(0, 0);
        };
        if (MODE == C2_MASK) mask_ld(0);
        for (int c = 0; c < cnt; c += ECH) {
          size_t pix;
          const bool ok = outpos(c, pix);
          uint2 mm[CPT / 4];
          if (MODE == C2_MASK) {
#pragma unroll
            for (int v4 = 0; v4 < CPT / 4; ++v4) mm[v4] = mn[v4];
            if (c + ECH < cnt) mask_ld(c + ECH);
          }
          uint32_t r[ECH];
          if (c + shift + ECH <= NT)
            tmem_ld16(tq + c + shift, r);
          else
            ld_tail13(tq + c + shift, r);
          tmem_ld_wait();
          float* dst = sPg + q * (ECH * SPS) + lane;   // sP[q][j][k], k = lane
#pragma unroll
          for (int j = 0; j < ECH; ++j) dst[j * SPS] = __uint_as_float(r[j]);
          named_bar(1 + grp, 128);
          {
            if (ok) {
#pragma unroll
              for (int v4 = 0; v4 < CPT / 4; ++v4) {
                float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int tp = 0; tp < TAPS; ++tp) {
                  const float4 a = *reinterpret_cast<const float4*>(sPg + (tp * QPT + cblk) * (ECH * SPS) + jj * SPS +
                                                                    cl + 4 * v4);
                  sum.x += a.x, sum.y += a.y, sum.z += a.z, sum.w += a.w;
                }
                const size_t off = pix * COUT + c0ch + 4 * v4;
                uint2 v;
                if (MODE == C2_MASK) {
                  const uint2 m2 = mm[v4];
                  v.x = pack_bf16x2(__uint_as_float(m2.x << 16) > 0.f ? sum.x : 0.f,
                                    __uint_as_float(m2.x & 0xffff0000u) > 0.f ? sum.y : 0.f);
                  v.y = pack_bf16x2(__uint_as_float(m2.y << 16) > 0.f ? sum.z : 0.f,
                                    __uint_as_float(m2.y & 0xffff0000u) > 0.f ? sum.w : 0.f);
                } else {
                  if (fullmap && bias) {
                    const float4 a = *reinterpret_cast<const float4*>(bias + pix % ((size_t)g.n1 * g.n2) * COUT + c0ch + 4 * v4);
                    sum.x += a.x, sum.y += a.y, sum.z += a.z, sum.w += a.w;
                  } else {
                    sum.x += bch[4 * v4], sum.y += bch[4 * v4 + 1], sum.z += bch[4 * v4 + 2], sum.w += bch[4 * v4 + 3];
                  }
                  v.x = pack_bf16x2(fmaxf(sum.x, 0.f), fmaxf(sum.y, 0.f));
                  v.y = pack_bf16x2(fmaxf(sum.z, 0.f), fmaxf(sum.w, 0.f));
                }
                *reinterpret_cast<uint2*>(h2 + off) = v;
              }
            }
          }
          named_bar(1 + grp, 128);
        }
        tc_fence_before();
        if (lane == 0) mbar_arrive(&tempty[buf]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync_all();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

static Geo make_geo(int batch, int n1, int n2, int R = C2_ROWS) {
  Geo g;
  g.n1 = n1, g.n2 = n2;
  g.wseg = n2 < WSEG ? n2 : WSEG;
  g.P = conv2_tc_box_cols(n2);
  g.nrb = (n1 + R - 1) / R;
  g.ncs = (n2 + g.wseg - 1) / g.wseg;
  g.units = batch * g.nrb * g.ncs;
  g.balanced = 1;
  g.batch = batch;
  g.ntall = 0;
  g.srows = R + 10;
  // the last row block goes to the end of the enumeration when its units run fewer tiles than the full ones
  const int Lfull = (std::min(R, n1) - 1) * g.P + g.wseg, rl = n1 - (g.nrb - 1) * R, Llast = (rl - 1) * g.P + g.wseg;
  g.nfull = (Lfull + OUT_PER_TILE - 1) / OUT_PER_TILE == (Llast + OUT_PER_TILE - 1) / OUT_PER_TILE ? g.nrb : g.nrb - 1;
  return g;
}

static int geo_tiles(const Geo& g) {   // MMA tiles of one image column segment
  int n = 0;
  for (int rb = 0; rb < g.nrb; ++rb) {
    const int r0 = rb * C2_ROWS + std::min(rb, g.ntall), rows = std::min(C2_ROWS + (rb < g.ntall), g.n1 - r0);
    int nt;
    tile_span(g, (rows - 1) * g.P + g.wseg, nt);
    n += nt;
  }
  return n;
}

// Mixed row-block heights (the R = 6, C_in = 64 layer-2 instance, one column segment): n1 = ntall (R + 1) +
// (nrb - ntall) R with nrb = ceil(n1 / (R + 1)) blocks, used when every block runs the same number of tiles and the
// image needs fewer tiles than with R-row blocks and a short last one.  Each tile restreams all 33 weight K-blocks
// (528 KB), and that stream bounds the kernel: at 64 x 64, 4 blocks of 7 rows (478 positions, tiles
// of 237 + 241) and 6 of 6 (2 x 205) are 20 tiles per image instead of 10 x 2 + 2 (the 4-row last block).
int conv2_tc_tall_blocks(int n1, int n2) {
  if (n2 > WSEG) return 0;
  const int nrb = (n1 + C2_ROWS) / (C2_ROWS + 1), ntall = n1 - C2_ROWS * nrb;
  if (ntall <= 0 || ntall > nrb) return 0;
  Geo a = make_geo(1, n1, n2), m = a;
  m.nrb = nrb, m.ntall = ntall;
  int ttall, tshort;
  tile_span(m, C2_ROWS * m.P + m.wseg, ttall);
  tile_span(m, (C2_ROWS - 1) * m.P + m.wseg, tshort);
  if (ttall != tshort) return 0;
  return geo_tiles(m) < geo_tiles(a) ? ntall : 0;
}
static Geo make_geo_c2(int batch, int n1, int n2, int mixed) {
  Geo g = make_geo(batch, n1, n2);
  const int nt = mixed ? conv2_tc_tall_blocks(n1, n2) : 0;
  if (nt > 0) {
    g.nrb = (n1 + C2_ROWS) / (C2_ROWS + 1);
    g.ntall = nt, g.srows = C2_ROWS + 11;
    g.units = batch * g.nrb * g.ncs;
    // every unit runs two tiles, so multicast pairs always consume the same K-blocks; they also keep the same pace
    // when a pair never straddles a tall and a short unit: with an even count of each per image the natural order
    // (image by image, row blocks top to bottom -- neighbouring CTAs share strip rows in L2) does that, otherwise the
    // tall units of all images go first
    g.nfull = (nt * g.ncs) % 2 == 0 && ((g.nrb - nt) * g.ncs) % 2 == 0 ? g.nrb : nt;
  }
  return g;
}

// Weight multicast across CTA pairs (MC) needs both CTAs of every pair to run the same number of tiles: an even
// grid, an even remainder of units over the grid, and the last row-block's units as many tiles as the full ones.
static bool pair_balanced(const Geo& g, int grid, int R, int cl = 2) {
  (void)R;   // full-tile units first (unit_of): the boundary to the shorter units must fall between clusters
  if (g.ntall > 0 && g.nfull == g.nrb && ((g.ntall * g.ncs) % cl != 0 || (g.nrb * g.ncs) % cl != 0))
    return false;   // mixed heights in natural order: clusters of cl units must not straddle a tall and a short unit
  return grid % cl == 0 && (g.units % grid) % cl == 0 && (g.batch * g.nfull * g.ncs) % cl == 0;
}
// And every pair must be co-resident: a GPC with an odd number of usable SMs cannot host a 2-CTA cluster on all of
// them, and a persistent grid whose last pair waits for a free GPC pair would take twice as long.  The occupancy
// query (once per kernel and shared-memory size) gates MC on all grid / 2 clusters fitting at once.
template <typename Kern>
static bool pairs_fit(Kern kern, int grid, int threads, size_t smem, int cl = 2) {
  struct Entry {
    const void* k;
    size_t smem;
    int grid, max;
  };
  static Entry cache[4] = {};
  static int ncache = 0;
  static std::mutex mu;   // contexts on several host threads
  std::lock_guard<std::mutex> lock(mu);
  for (int i = 0; i < ncache; ++i)
    if (cache[i].k == (const void*)kern && cache[i].smem == smem && cache[i].grid == grid) return cl * cache[i].max >= grid;
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid), cfg.blockDim = dim3(threads), cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl, at[0].val.clusterDim.y = 1, at[0].val.clusterDim.z = 1;
    cfg.attrs = at, cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
      (void)cudaGetLastError();
      n = 0;
    }
    cache[ncache < 4 ? ncache++ : 3] = Entry{(const void*)kern, smem, grid, n};
    if (getenv("DI_DEBUG_MC")) fprintf(stderr, "conv2: %d co-resident clusters of %d (grid %d)\n", n, cl, grid);
    return cl * n >= grid;
  }
}
// cluster launch, programmatic dependent launch (the kernel waits for its predecessor in griddep_wait)
template <typename... Args>
static cudaError_t launch_pair(void (*kern)(Args...), int grid, int threads, size_t smem, cudaStream_t st,
                               const CUtensorMap& tm, const __nv_bfloat16* w, const float* bias, int fullmap, Geo g,
                               __nv_bfloat16* out, const __nv_bfloat16* mask, int cl = 2) {
  return launch_ex(kern, dim3(grid), dim3(threads), smem, st, cl, true, tm, w, bias, fullmap, g, out, mask);
}

// room for the R + 11-row strip of mixed heights whenever they may apply (one column segment)
size_t conv2_tc_smem_bytes(int n2) {
  const int P = conv2_tc_box_cols(n2);
  const int rows = R + 10 + (n2 <= WSEG ? 1 : 0);
  const size_t strip_alloc = ((size_t)strip_rows_bytes(rows, P) + GUARD_ROWS * 128 + 1023) & ~(size_t)1023;
  return strip_alloc + WSTAGES * WBYTES + 4 * ECH * SPS * 4 + 1024;
}
// <32, 64, C2_MASK>: strip of 64-B rows, C2_WST64 weight stages of 8 KB, two epilogue groups
static size_t dgrad2_bf16_smem_bytes(int n2) {
  const int wseg = n2 < WSEG ? n2 : WSEG, P = wseg + 10;
  const size_t strip_alloc = ((size_t)(C2_DG_ROWS + 10) * P * 64 + GUARD_ROWS * 64 + 1023) & ~(size_t)1023;
  return strip_alloc + (size_t)C2_WST64 * 8192 + 2 * 4 * ECH * SPS * 4 + 1024;
}

// The strip is loaded in one box per unit.  Loading it as two halves with a separate producer so that the load
// overlaps the MMAs of the previous unit removes the strip wait but measured slower on B200 (the TMA writes
// compete with the UMMA operand reads for shared-memory bandwidth, which this kernel saturates: DESIGN.md §11).
int conv2_tc_box_rows(int n1, int n2, int mixed) { return R + 10 + (mixed && conv2_tc_tall_blocks(n1, n2) > 0); }
int dgrad2_bf16_box_rows() { return C2_DG_ROWS + 10; }
// Strip pitch P (positions per strip row).  One column segment (n2 <= 64): P = n2 + 5 -- the box starts 5 columns
// left of the image, so its 5 out-of-bounds (zero) columns are the left padding of a row AND the right padding of the
// row above (a tap window c + v - 5 >= n2 runs into the next strip row's zero columns).  Several segments: the
// halos are image data on both sides, P = 64 + 10.  P = 69 instead of 74 cuts the MMA columns per 6 x 64 output
// block from 448 to 416; measured on B200 (same box, alternating): conv2 6.62 vs 6.75 ms (+1.7 %) -- the kernel
// is bound by the shared-memory port, not by the MMA columns.
int conv2_tc_box_cols(int n2) { return n2 <= WSEG ? n2 + 5 : WSEG + 10; }

cudaError_t setup_conv2_tc(int n2) {
  cudaError_t e = cudaFuncSetAttribute(k_conv2_tc<64, 32, C2_BIAS_RELU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)conv2_tc_smem_bytes(n2));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_conv2_tc<64, 32, C2_BIAS_RELU, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)conv2_tc_smem_bytes(n2));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_conv2_tc<64, 32, C2_BIAS_RELU, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)conv2_tc_smem_bytes(n2));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_conv2_tc<32, 64, C2_MASK, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)dgrad2_bf16_smem_bytes(n2));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_conv2_tc<32, 64, C2_MASK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)dgrad2_bf16_smem_bytes(n2));
}

// cluster: weight-multicast cluster size (the context's setting, read once by di_create: 2 by default, DI_EXP_NO_MC=1
// -> 1, DI_EXP_C2_CLUSTER=4 -> 4); falls back to smaller clusters when the balance / co-residency checks fail
cudaError_t launch_conv2_tc(const CUtensorMap* tmH1, const void* wpack, const float* bias, int fullmap, int batch,
                            int n1, int n2, void* h2, int num_sms, cudaStream_t st, int cluster, int balanced,
                            int mixed) {
  Geo g = make_geo_c2(batch, n1, n2, mixed);
  g.balanced = balanced;
  const int grid = g.units < num_sms ? g.units : num_sms;
  const size_t sm = conv2_tc_smem_bytes(n2);
  const __nv_bfloat16* w = reinterpret_cast<const __nv_bfloat16*>(wpack);
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(h2);
  if (cluster >= 4 && pair_balanced(g, grid, R, 4) && pairs_fit(k_conv2_tc<64, 32, C2_BIAS_RELU, 4>, grid, 256, sm, 4))
    return launch_pair(k_conv2_tc<64, 32, C2_BIAS_RELU, 4>, grid, 256, sm, st, *tmH1, w, bias, fullmap, g, out,
                       (const __nv_bfloat16*)nullptr, 4);
  if (cluster >= 2 && pair_balanced(g, grid, R) && pairs_fit(k_conv2_tc<64, 32, C2_BIAS_RELU, 2>, grid, 256, sm))
    return launch_pair(k_conv2_tc<64, 32, C2_BIAS_RELU, 2>, grid, 256, sm, st, *tmH1, w, bias, fullmap, g, out,
                       (const __nv_bfloat16*)nullptr);
  return launch_pair(k_conv2_tc<64, 32, C2_BIAS_RELU>, grid, 256, sm, st, *tmH1, w, bias, fullmap, g, out,
                     (const __nv_bfloat16*)nullptr, 1);
}

// custom stacks, BF16 contexts: interior C_in -> C_out layers (C in {32, 64}) on the same
// kernel, weights packed by convg_tc_pack (K-block u * J + j, rows v' * C_out + k, C_in bf16 channels per row).
// tm: bf16 strip map over the input activation (box C_in x P x convg_tc_box_rows(C_in)); out: NHWC, C_out channels.
int convg_tc_box_rows(int cin) { return (cin >= 64 ? C2_ROWS : C2_DG_ROWS) + 10; }

// <64, 64>: the 128-B-row strip, a 3-stage ring and two epilogue groups' staging
static size_t convg64_smem_bytes(int n2) {
  const int P = conv2_tc_box_cols(n2);
  const size_t strip_alloc = ((size_t)strip_rows_bytes(R + 10, P) + GUARD_ROWS * 128 + 1023) & ~(size_t)1023;
  return strip_alloc + 3 * WBYTES + 2 * 4 * ECH * SPS * 4 + 1024;
}

template <int CIN, int COUT>
static size_t convg_smem(int n2) {
  return CIN == 32 ? dgrad2_bf16_smem_bytes(n2) : COUT >= 64 ? convg64_smem_bytes(n2) : conv2_tc_smem_bytes(n2);
}
template <int CIN, int COUT>
static cudaError_t launch_g(const CUtensorMap* tm, const void* wpack, const float* bias, int batch, int n1, int n2,
                            void* out, int num_sms, cudaStream_t st) {
  Geo g = make_geo(batch, n1, n2, CIN >= 64 ? C2_ROWS : C2_DG_ROWS);
  const int grid = g.units < num_sms ? g.units : num_sms;
  k_conv2_tc<CIN, COUT, C2_BIAS_RELU><<<grid, COUT >= 64 ? 384 : 256, convg_smem<CIN, COUT>(n2), st>>>(
      *tm, reinterpret_cast<const __nv_bfloat16*>(wpack), bias, 0, g, reinterpret_cast<__nv_bfloat16*>(out), nullptr);
  return cudaGetLastError();
}

template <int CIN, int COUT>
static cudaError_t setup_g(int n2) {
  return cudaFuncSetAttribute(k_conv2_tc<CIN, COUT, C2_BIAS_RELU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)convg_smem<CIN, COUT>(n2));
}

cudaError_t setup_convg_tc(int n2) {
  cudaError_t e;
  if ((e = setup_g<64, 128>(n2)) != cudaSuccess || (e = setup_g<128, 64>(n2)) != cudaSuccess ||
      (e = setup_g<128, 32>(n2)) != cudaSuccess || (e = setup_g<128, 128>(n2)) != cudaSuccess ||
      (e = setup_g<32, 128>(n2)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(k_conv2_tc<64, 64, C2_BIAS_RELU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)convg64_smem_bytes(n2))) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(k_conv2_tc<32, 32, C2_BIAS_RELU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)dgrad2_bf16_smem_bytes(n2))) != cudaSuccess)
    return e;
  return cudaFuncSetAttribute(k_conv2_tc<32, 64, C2_BIAS_RELU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)dgrad2_bf16_smem_bytes(n2));
}

cudaError_t launch_convg_tc(int cin, int cout, const CUtensorMap* tm, const void* wpack, const float* bias, int batch,
                            int n1, int n2, void* out, int num_sms, cudaStream_t st) {
  if (cin == 64 && cout == 32) return launch_g<64, 32>(tm, wpack, bias, batch, n1, n2, out, num_sms, st);
  if (cin == 64 && cout == 64) return launch_g<64, 64>(tm, wpack, bias, batch, n1, n2, out, num_sms, st);
  if (cin == 32 && cout == 32) return launch_g<32, 32>(tm, wpack, bias, batch, n1, n2, out, num_sms, st);
  if (cin == 32 && cout == 64) return launch_g<32, 64>(tm, wpack, bias, batch, n1, n2, out, num_sms, st);
  if (cin == 64 && cout == 128) return launch_g<64, 128>(tm, wpack, bias, batch, n1, n2, out, num_sms, st);
  if (cin == 128 && cout == 64) return launch_g<128, 64>(tm, wpack, bias, batch, n1, n2, out, num_sms, st);
  if (cin == 128 && cout == 32) return launch_g<128, 32>(tm, wpack, bias, batch, n1, n2, out, num_sms, st);
  if (cin == 128 && cout == 128) return launch_g<128, 128>(tm, wpack, bias, batch, n1, n2, out, num_sms, st);
  if (cin == 32 && cout == 128) return launch_g<32, 128>(tm, wpack, bias, batch, n1, n2, out, num_sms, st);
  return cudaErrorInvalidValue;
}

// training: the layer-2 data gradient on the bf16 layer-2 machinery (TMEM double buffering, weights per tile):
// tmDGb = dG2 [B][n1][n2][32] bf16 strips (box 32 ch x P x (C2_DG_ROWS + 10) rows, SWIZZLE_64B), wpack = 66 x 8-KB blocks
// (rows v' * 64 + ci, 32 co, SWIZZLE_64B), h1b = bf16 h1 (the ReLU' mask), dh1b = bf16 output
cudaError_t launch_dgrad2_bf16(const CUtensorMap* tmDGb, const void* wpack, const void* h1b, int batch, int n1, int n2,
                               void* dh1b, int num_sms, cudaStream_t st) {
  Geo g = make_geo(batch, n1, n2, C2_DG_ROWS);
  const int grid = g.units < num_sms ? g.units : num_sms;
  if (pair_balanced(g, grid, C2_DG_ROWS) &&
      pairs_fit(k_conv2_tc<32, 64, C2_MASK, 2>, grid, 384, dgrad2_bf16_smem_bytes(n2)))
    return launch_pair(k_conv2_tc<32, 64, C2_MASK, 2>, grid, 384, dgrad2_bf16_smem_bytes(n2), st, *tmDGb,
                       reinterpret_cast<const __nv_bfloat16*>(wpack), nullptr, 0, g,
                       reinterpret_cast<__nv_bfloat16*>(dh1b), reinterpret_cast<const __nv_bfloat16*>(h1b));
  k_conv2_tc<32, 64, C2_MASK><<<grid, 384, dgrad2_bf16_smem_bytes(n2), st>>>(
      *tmDGb, reinterpret_cast<const __nv_bfloat16*>(wpack), nullptr, 0, g, reinterpret_cast<__nv_bfloat16*>(dh1b),
      reinterpret_cast<const __nv_bfloat16*>(h1b));
  return cudaGetLastError();
}

DI_DEBUG_BINDER(di_debug_bind_k_conv2_tc)

}  // namespace di
