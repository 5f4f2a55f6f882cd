// k_conv3_r4.cu -- stage 3 of the bf16 path, conv layer 3 (1 filter 11x11x32 + bias, ReLU iff DI_FLAG_FINAL_RELU,
// crop S) with RP = 11 OUTPUT ROWS STACKED IN M.
//
// C_out = 1 leaves the UMMA M dimension to the taps.  The first design (k_conv3_tc) stacks the 11 column taps of one
// tap row in M = 32 (.ws) and walks the 11 tap rows as K-blocks, so every strip position is read by 11 MMAs per
// 246 outputs and the tensor core's shared-memory reads bound it (0.87 ms at lowrate).  Here M = 128 holds RP = 11
// output rows t x ES = 11 rows (the column taps v; 121 of the 128 rows used): window k (k = 0 .. RP + 9) is the strip
// shifted by k rows, and rows (t, .) of its A operand hold the taps of tap row u = k - t, so that
//   D[(t, v)][n] = sum_k sum_c W[k - t][v][c] strip[n + k P][c]  and  x_hat[row t][j] = sum_v D[(t, v)][j + v].
// A_k = [W[k]; W[k-1]; ...; W[k-RP+1]] is a 128-row window of ONE stack T[i] = W[10 - i] (zero outside 0..10): A_k
// starts at T[10 - k] (an 11-row entry: any 64-B row may start a SWIZZLE_64B window, tools/ladder.cu t3/t11), the
// whole bank stays resident in shared memory, and a window is a descriptor start address.  N = P rounded up to 16
// (<= 80) covers one strip row: per 11 x 64 outputs 21 windows x 2 MMAs (K = 16) -- 0.060 MMAs per output against
// 0.070 with 8 rows x 16-row entries (r02: 0.40 ms) and 0.09 for k_conv3_tc.  The 121 tap rows do not align with
// the TMEM lane quadrants, so the four epilogue warps share one tile (see the epilogue).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>

#include "kernels.cuh"
#define DI_TU_ID 4
#include "sm100.cuh"

namespace di {

namespace {
constexpr int RP = C3R_RP, ES = C3R_ES, NWIN = C3R_NWIN, IMIN = C3R_IMIN;
constexpr int R = RP;                  // output rows per unit (one pass)
constexpr int CH = R;                  // strip rows per TMA chunk (chunk k = strip rows [R k - 5, R k + R - 5))
constexpr int NSPAN = (R + 10 + CH - 1) / CH;   // chunks a unit reads (R + 10 strip rows): 2 for R = 11
constexpr int NCH = NSPAN + 1;         // chunk slots in the ring: one loads while a unit computes
constexpr int NACC = 4;                // TMEM accumulator slots (128 columns each)
#ifndef DI_C3R_PF
#define DI_C3R_PF 6
#endif
constexpr int C3R_PF = DI_C3R_PF;      // chunks prefetched into L2 ahead of the shared-memory loads
constexpr int TBLK = ES * 64;          // one T entry: ES rows (v) x 32 channels bf16, SWIZZLE_64B
constexpr int TBYTES = (C3R_NENT * TBLK + 1023) & ~1023;
constexpr int GUARD = 16;              // zero positions past the ring (the last ring row's window reads N - P past it)
constexpr int SROW = 84;               // epilogue tile row stride (floats): 16-B rows
constexpr int SROWS = RP * ES;         // TMEM lanes holding taps (121 of 128 for RP = ES = 11)
constexpr int OPT = (RP * 64 + 127) / 128;   // outputs per epilogue thread and unit

// Work item = one column segment of one image (or a contiguous part of its row blocks when there are fewer
// columns than SMs): its units run top to bottom, so consecutive units share 10 of their 18 strip rows.
struct GeoR4 {
  int n1, n2, wseg, P, N, nrb, ncs, splits, per, items;
};
__device__ __forceinline__ void item_of(const GeoR4& g, int it, int& b, int& c0, int& rb0, int& nu) {
  const int col = it / g.splits, sp = it - col * g.splits;
  b = col / g.ncs;
  c0 = (col - b * g.ncs) * g.wseg;
  rb0 = sp * g.per;
  nu = min(g.per, g.nrb - rb0);
}
}  // namespace

// Strip rows arrive in chunks of CH = 8 rows through a ring of NCH = 4 chunk slots (ROW RING): unit j of an item
// (output rows 8 (rb0 + j) .. + 7) reads strip rows [8 (rb0 + j) - 5, + 18) = chunks j, j + 1, j + 2 of the item, and
// releases chunk j when its MMAs complete, so chunk j + 3 loads while unit j computes.  Each strip row is fetched
// once per item (10 chunks = 80 rows for a 64-row image) instead of 18 rows per 8-row unit: the L2 -> shared-memory
// traffic drops from 2.25x to 1.25x the h2 rows.  Window k of a unit reads ring row (8 (chunk j) + k) mod 32 plus
// N - P positions past it (the next row, the slot padding or the zero guard); those positions only reach D columns
// >= P, which no output reads.
//
// Fused metrics (di_recover_metrics): with xtrue != null each epilogue thread also reads the
// ground truth of the outputs it writes and accumulates, in fp64 and a fixed order, sum (x_hat - x)^2, sum x^2 and
// max x; per item the four warps' sums go to mpart[item][warp][3] (no atomics), and k_metrics_finish combines the
// items of each image in item order: PSNR, NMSE and success without a second pass over
// x_hat.
template <bool METRICS>
__global__ void __launch_bounds__(256, 1)
    k_conv3_r4(const __grid_constant__ CUtensorMap tmH2, const uint8_t* __restrict__ tpack,
               const float* __restrict__ bias, int fullmap, int relu, GeoR4 g, float* __restrict__ xhat,
               const float* __restrict__ xtrue, double* __restrict__ mpart) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int P = g.P;
  const int chunk_bytes = CH * P * 64;
  const int slot = (chunk_bytes + 1023) & ~1023;              // slot stride: 1024-aligned TMA destinations
  uint8_t* const tb = smem;                                   // T stack (1024-aligned)
  uint8_t* const ring = smem + TBYTES;                        // NCH chunk slots, then the zero guard
  const int ring_alloc = (NCH * slot + GUARD * 64 + 1023) & ~1023;
  float* const S = reinterpret_cast<float*>(ring + ring_alloc);

  __shared__ uint64_t wbar, cfull[NCH], cempty[NCH], acc_full[NACC], acc_empty[NACC];
  __shared__ uint32_t tslot;
  const int warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmH2);
    mbar_init(&wbar, 1);
    for (int s = 0; s < NCH; ++s) mbar_init(&cfull[s], 1), mbar_init(&cempty[s], 1);
    for (int a = 0; a < NACC; ++a) mbar_init(&acc_full[a], 1), mbar_init(&acc_empty[a], 4);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&tslot), tmem_relinquish();
  for (int i = threadIdx.x; i < ring_alloc / 16; i += blockDim.x)   // finite ring (never-loaded slots) and guard
    reinterpret_cast<uint4*>(ring)[i] = make_uint4(0, 0, 0, 0);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ producer: T once, strip chunks
      mbar_arrive_expect_tx(&wbar, TBYTES);
      bulk_load(tb, tpack, TBYTES, &wbar);
      // L2 prefetch cursor, PF chunks ahead of the loads: the ring holds one chunk of lead (one unit of MMAs), too
      // few bytes in flight to cover DRAM latency; the prefetched chunks arrive from L2
      int pit = blockIdx.x, pk = 0, pb = 0, pc0 = 0, prb0 = 0, pnu = 0;
      if (pit < g.items) item_of(g, pit, pb, pc0, prb0, pnu);
      auto prefetch_next = [&]() {
        if (pit >= g.items) return;
        tma_prefetch_l2_4d(&tmH2, 0, pc0 - 5, CH * (prb0 + pk) - 5, pb);
        if (++pk == pnu + NSPAN - 1) {
          pk = 0, pit += gridDim.x;
          if (pit < g.items) item_of(g, pit, pb, pc0, prb0, pnu);
        }
      };
      for (int i = 0; i < C3R_PF; ++i) prefetch_next();
      uint32_t gc = 0;                 // chunks issued by this CTA
      for (int it = blockIdx.x; it < g.items; it += gridDim.x) {
        int b, c0, rb0, nu;
        item_of(g, it, b, c0, rb0, nu);
        for (int k = 0; k < nu + NSPAN - 1; ++k, ++gc) {
          const uint32_t sl = gc % NCH;
          if (gc >= NCH) mbar_wait(&cempty[sl], ((gc / NCH) - 1) & 1);
          mbar_arrive_expect_tx(&cfull[sl], chunk_bytes);
          tma_load_4d(ring + sl * slot, &tmH2, &cfull[sl], 0, c0 - 5, CH * (rb0 + k) - 5, b);
          prefetch_next();
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      mbar_wait(&wbar, 0);
      tc_fence_after();
      const uint32_t idesc = idesc_f32acc(1, 128, g.N);
      const uint64_t adesc0 = smem_desc(smem_u32(tb), 16, 512, kSwizzle64B);
      const uint64_t bdesc0 = smem_desc(smem_u32(ring), 16, 512, kSwizzle64B);
      const uint64_t rstep = (uint64_t)((P * 64) >> 4);                  // one strip row
      const uint64_t padstep = (uint64_t)((slot - chunk_bytes) >> 4);     // slot padding after a slot's last row
      const uint64_t ringstep = (uint64_t)((NCH * slot) >> 4);           // the whole ring
      uint32_t gc0 = 0;                // this item's first chunk (CTA-wide count)
      int pi = 0;
#ifdef DI_PROF_CONV3
      long long pc_chunk = 0, pc_acc = 0, pc0 = clock64(), pt;
#define C3P0 pt = clock64();
#define C3P1(acc) acc += clock64() - pt;
#else
#define C3P0
#define C3P1(acc)
#endif
      for (int it = blockIdx.x; it < g.items; it += gridDim.x) {
        int b, c0, rb0, nu;
        item_of(g, it, b, c0, rb0, nu);
        for (int k = 0; k < NSPAN - 1; ++k) {   // the item's first chunks
          const uint32_t c = gc0 + k;
          C3P0 mbar_wait(&cfull[c % NCH], (c / NCH) & 1); C3P1(pc_chunk)
        }
        for (int j = 0; j < nu; ++j, ++pi) {
          const uint32_t cj = gc0 + j;
          C3P0 mbar_wait(&cfull[(cj + NSPAN - 1) % NCH], ((cj + NSPAN - 1) / NCH) & 1); C3P1(pc_chunk)
          tc_fence_after();
          const int a = pi % NACC;
          if (pi >= NACC) {
            C3P0 mbar_wait(&acc_empty[a], ((pi / NACC) - 1) & 1); C3P1(pc_acc)
            tc_fence_after();
          }
          const uint32_t d = tmem + a * 128;
          const int sl0 = (int)(cj % NCH);                     // slot of the unit's strip row 0
          // a window reads N - P positions past its row: the last slot's last row runs into the zero guard
          DI_DEVICE_ASSERT(g.N - g.P <= GUARD, g.N, g.P);
          // the single issuing thread is latency-bound: the B descriptor advances by adds only (one strip row per
          // window, the slot padding every CH rows, back to slot 0 after the last slot)
          uint64_t bd = bdesc0 + (uint64_t)((sl0 * slot) >> 4);
          const int kwrap = (NCH - sl0) * CH - 1;               // last window before the ring wraps
#pragma unroll
          for (int k = 0; k < NWIN; ++k) {
            const uint64_t ad = adesc0 + (uint64_t)(((10 - k - IMIN) * TBLK) >> 4);   // T[10 - k] ..
            umma_f16_ss(d, ad, bd, idesc, k != 0);
            umma_f16_ss(d, ad + 2, bd + 2, idesc, 1);                       // channels 16..31: +32 B
            bd += rstep;
            if ((k % CH) == CH - 1) bd += padstep;
            if (k == kwrap) bd -= ringstep;
          }
          umma_commit(&acc_full[a]);
          umma_commit(&cempty[cj % NCH]);                     // chunk j is read by units j - NSPAN + 1 .. j only
        }
        for (int k = 0; k < NSPAN - 1; ++k) umma_commit(&cempty[(gc0 + nu + k) % NCH]);   // the item's last chunks
        gc0 += nu + NSPAN - 1;
      }
#ifdef DI_PROF_CONV3
      if (blockIdx.x % 37 == 0)
        printf("conv3 cta %d issuer: cycles %lld chunk-wait %lld acc-wait %lld units %d\n", blockIdx.x,
               clock64() - pc0, pc_chunk, pc_acc, pi);
#endif
    }
  } else if (warp >= 4) {  // ---------------------------------------------------------------------- epilogue
    // The RP x ES tap rows do not align with the 32-lane TMEM quadrants (ES = 11), so the four warps write their
    // quadrants into ONE shared tile S[lane][column] and then sum the 11 diagonals of every output from it:
    // x_hat[row t][j] = sum_v S[t ES + v][j + v] -- 128 threads, consecutive j per warp (conflict-free).
    const int q = warp - 4, e = threadIdx.x - 128;
    const float bsc = (!fullmap && bias) ? bias[0] : 0.f;
    int pi = 0;
    for (int it = blockIdx.x; it < g.items; it += gridDim.x) {
      int b, c0, rb0, nu;
      item_of(g, it, b, c0, rb0, nu);
      double m_se = 0.0, m_sx = 0.0;
      float m_mx = -INFINITY;
      for (int j = 0; j < nu; ++j, ++pi) {
        const int r0 = (rb0 + j) * R;
        const int a = pi % NACC;
        // METRICS: the ground truth of this thread's outputs, loaded before the accumulator wait so the global-load
        // latency overlaps it
        float tv[OPT];
        if (METRICS) {
#pragma unroll
          for (int h = 0; h < OPT; ++h) {
            const int idx = e + 128 * h, t = idx >> 6, jc = idx & 63, row = r0 + t;
            tv[h] = (idx < RP * 64 && jc < g.wseg && c0 + jc < g.n2 && row < g.n1)
                        ? __ldg(xtrue + ((size_t)b * g.n1 + row) * g.n2 + c0 + jc) : 0.f;
          }
        }
        mbar_wait(&acc_full[a], (pi / NACC) & 1);
        tc_fence_after();
        const uint32_t taddr = tmem + a * 128 + ((uint32_t)(q * 32) << 16);
        uint32_t r[80];
        tmem_ld32(taddr, r);
        tmem_ld32(taddr + 32, r + 32);
        tmem_ld16(taddr + 64, r + 64);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[a]);
        named_bar(1, 128);          // the previous unit's sums are done with S
        const int L = q * 32 + lane;
        if (L < SROWS) {
          float4* dst = reinterpret_cast<float4*>(S + L * SROW);
#pragma unroll
          for (int jj = 0; jj < 20; ++jj)
            dst[jj] = make_float4(__uint_as_float(r[4 * jj]), __uint_as_float(r[4 * jj + 1]),
                                  __uint_as_float(r[4 * jj + 2]), __uint_as_float(r[4 * jj + 3]));
        }
        named_bar(1, 128);          // S holds every tap row of this unit
#pragma unroll
        for (int h = 0; h < OPT; ++h) {
          const int idx = e + 128 * h, t = idx >> 6, jc = idx & 63;
          if (idx >= RP * 64) break;
          const int row = r0 + t;
          const float* sr = S + t * ES * SROW + jc;
          float acc = 0.f;
#pragma unroll
          for (int v = 0; v < 11; ++v) acc += sr[v * SROW + v];
          if (jc < g.wseg && c0 + jc < g.n2 && row < g.n1) {
            const size_t pix = ((size_t)b * g.n1 + row) * g.n2 + c0 + jc;
            acc += (fullmap && bias) ? bias[pix % ((size_t)g.n1 * g.n2)] : bsc;
            if (relu) acc = fmaxf(acc, 0.f);
            xhat[pix] = acc;
            if (METRICS) {
              const float tt = tv[h];
              const double dd = (double)acc - (double)tt;
              m_se += dd * dd, m_sx += (double)tt * (double)tt, m_mx = fmaxf(m_mx, tt);
            }
          }
        }
      }
      if (METRICS) {   // the warp's sums for this item, butterfly order fixed
        for (int o = 16; o > 0; o >>= 1) {
          m_se += __shfl_xor_sync(0xffffffffu, m_se, o);
          m_sx += __shfl_xor_sync(0xffffffffu, m_sx, o);
          m_mx = fmaxf(m_mx, __shfl_xor_sync(0xffffffffu, m_mx, o));
        }
        if (lane == 0) {
          double* mp = mpart + ((size_t)it * 4 + q) * 3;
          mp[0] = m_se, mp[1] = m_sx, mp[2] = (double)m_mx;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

static GeoR4 make_geo_r4(int batch, int n1, int n2, int num_sms) {
  GeoR4 g;
  g.n1 = n1, g.n2 = n2;
  g.wseg = n2 < 64 ? n2 : 64;
  g.P = g.wseg + 10;
  g.N = (g.P + 15) & ~15;
  g.nrb = (n1 + R - 1) / R;
  g.ncs = (n2 + g.wseg - 1) / g.wseg;
  const int cols = batch * g.ncs;
  // fewer columns than SMs: split each column into parts of `per` row blocks
  g.splits = cols >= num_sms ? 1 : std::min(g.nrb, (num_sms + cols - 1) / cols);
  g.per = (g.nrb + g.splits - 1) / g.splits;
  g.splits = (g.nrb + g.per - 1) / g.per;
  g.items = cols * g.splits;
  return g;
}

static size_t smem_r4(int n2) {
  const int wseg = n2 < 64 ? n2 : 64, P = wseg + 10;
  const size_t slot = ((size_t)CH * P * 64 + 1023) & ~(size_t)1023;
  const size_t ring_alloc = (NCH * slot + GUARD * 64 + 1023) & ~(size_t)1023;
  return TBYTES + ring_alloc + (size_t)SROWS * SROW * 4 + 1024;
}

int conv3_r4_box_rows() { return CH; }
int conv3_r4_tpack_bytes() { return TBYTES; }

cudaError_t setup_conv3_r4(int n2) {
  const cudaError_t e = cudaFuncSetAttribute(k_conv3_r4<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem_r4(n2));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_conv3_r4<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_r4(n2));
}

// per image b: the items b * per_img .. (b + 1) * per_img - 1, four warps each, summed in that order
__global__ void k_metrics_finish(const double* __restrict__ mpart, int per_img, int N, int batch,
                                 double* __restrict__ out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  double se = 0.0, sx = 0.0, mx = -INFINITY;
  const double* p = mpart + (size_t)b * per_img * 4 * 3;
  for (int i = 0; i < per_img * 4; ++i) se += p[3 * i], sx += p[3 * i + 1], mx = fmax(mx, p[3 * i + 2]);
  const double mse = se / N;
  out[b] = mse == 0.0 ? INFINITY : 10.0 * log10(mx * mx / mse);
  const double nmse = se / sx;
  out[batch + b] = nmse;
  out[2 * batch + b] = nmse <= 0.1 ? 1.0 : 0.0;
}

size_t conv3_r4_metrics_part_bytes(int batch, int n1, int n2, int num_sms) {
  const GeoR4 g = make_geo_r4(batch, n1, n2, num_sms);
  return (size_t)g.items * 4 * 3 * sizeof(double);
}

cudaError_t launch_conv3_r4(const CUtensorMap* tmH2, const void* tpack, const float* bias, int fullmap, int relu,
                            float* xhat, int batch, int n1, int n2, int num_sms, cudaStream_t st, const float* xtrue,
                            double* mpart, double* metrics) {
  GeoR4 g = make_geo_r4(batch, n1, n2, num_sms);
  const int grid = g.items < num_sms ? g.items : num_sms;
  if (xtrue)
    k_conv3_r4<true><<<grid, 256, smem_r4(n2), st>>>(*tmH2, reinterpret_cast<const uint8_t*>(tpack), bias, fullmap,
                                                    relu, g, xhat, xtrue, mpart);
  else
    k_conv3_r4<false><<<grid, 256, smem_r4(n2), st>>>(*tmH2, reinterpret_cast<const uint8_t*>(tpack), bias, fullmap,
                                                     relu, g, xhat, nullptr, nullptr);
  if (xtrue) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_metrics_finish<<<(batch + 127) / 128, 128, 0, st>>>(mpart, g.ncs * g.splits, n1 * n2, batch, metrics);
  }
  return cudaGetLastError();
}

DI_DEBUG_BINDER(di_debug_bind_k_conv3_r4)

}  // namespace di
