// k_conv3_r4.cu -- stage 3 of the bf16 path, conv layer 3 (1 filter 11x11x32 + bias, ReLU iff DI_FLAG_FINAL_RELU,
// crop S) with RP = 11 OUTPUT ROWS STACKED IN M, TWO IMAGES SIDE BY SIDE IN N, and the strip
// STREAMED ROW BY ROW.
//
// C_out = 1 leaves the UMMA M dimension to the taps.  The first design (k_conv3_tc) stacks the 11 column taps of one
// tap row in M = 32 (.ws) and walks the 11 tap rows as K-blocks, so every strip position is read by 11 MMAs per
// 246 outputs and the tensor core's shared-memory reads bound it (0.87 ms at lowrate).  Here M = 128 holds RP = 11
// output rows t x ES = 11 rows (the column taps v; 121 of the 128 rows used): window k (k = 0 .. RP + 9) of a unit is
// its strip row k, and rows (t, .) of its A operand hold the taps of tap row u = k - t, so that
//   D[(t, v)][n] = sum_k sum_c W[k - t][v][c] strip[row k][n][c]  and  x_hat[row t][j] = sum_v D[(t, v)][j + v].
// A_k = [W[k]; W[k-1]; ...; W[k-RP+1]] is a 128-row window of ONE stack T[i] = W[10 - i] (zero outside 0..10): A_k
// starts at T[10 - k] (an 11-row entry: any 64-B row may start a SWIZZLE_64B window, tools/ladder.cu t3/t11), the
// whole bank stays resident in shared memory, and a window is a descriptor start address.
//
// r02 (this version): a strip row holds the same image row of TWO images, PP = roundup16(W + 10) positions each
// (one 4-D TMA box over (channel, column, image, row)), so one MMA has N = 2 PP = 160 columns at 64 x 64 -- the
// A-operand read (4 KB per MMA, the cost that bound the one-image form at N = 80) is shared by twice the outputs.
// Three such rows would not fit the chunk ring of whole 21-row unit strips, so the strip is streamed instead: units
// j (output rows 11 j ..) overlap by 10 strip rows, and every strip row s feeds the (at most two) units that read
// it -- window s - 11 j + 5 of unit j -- in the same pass.  Each row is then consumed once and released: the ring
// only holds the lead (NSL rows), two units accumulate at a time (the third TMEM slot drains in the epilogue), and rows
// outside the image (the 5 zero rows above / below) are never loaded or multiplied.  The single issuing thread is
// latency-bound (a general per-row loop -- unit indices, modulo slot arithmetic -- ran at ~230 cycles per MMA), so
// rows are walked in groups of 11 aligned to the units (group jg: strip rows 11 jg - 5 + ka, ka = 0..10, feed unit
// jg at window ka and unit jg - 1 at window ka + 11): per group the accumulators, first / last flags and clipping
// are fixed, and the unrolled row loop is descriptor adds, one ring-slot wait and one commit per row.
// Per 2 x 64 x 64 outputs: 114 windows x 2 MMAs of N = 160 against 2 x 126 x 2 of N = 80.
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
constexpr int R = RP;                  // output rows per unit
constexpr int CHR = 1;                 // strip rows per TMA chunk (= ring slot)
#ifndef DI_C3R_NSL
#define DI_C3R_NSL 12
#endif
constexpr int NSL = DI_C3R_NSL;        // ring slots (rows of lead)
constexpr int NACC = 3;                // TMEM accumulator slots: two units accumulate, one drains
constexpr int ACOLS = 160;             // TMEM columns per slot (N <= 160)
#ifndef DI_C3R_PF
#define DI_C3R_PF 0
#endif
// rows prefetched into L2 ahead of the shared-memory loads (experiment builds): r04 measured the kernel 4 % faster
// without the prefetches (0.300 vs 0.305-0.314 ms; the issuer's row waits unchanged), so the product issues none
constexpr int C3R_PF = DI_C3R_PF;
constexpr int TBLK = ES * 64;          // one T entry: ES rows (v) x 32 channels bf16, SWIZZLE_64B
constexpr int TBYTES = (C3R_NENT * TBLK + 1023) & ~1023;
constexpr int SROW = 84;               // epilogue tile row stride (floats): 16-B rows
constexpr int SROWS = RP * ES;         // TMEM lanes holding taps (121 of 128 for RP = ES = 11)
constexpr int OPT = (RP * 64 + 127) / 128;   // outputs per epilogue thread, unit and image

// Work item = one column segment of one PAIR of images (2 p, 2 p + 1), or a contiguous part of its row blocks when
// there are fewer pair-columns than SMs.  Its strip rows s_lo .. s_hi - 1 stream top to bottom.
struct GeoR4 {
  int n1, n2, batch, wseg, PP, N, nrb, ncs, splits, per, items;
};
__device__ __forceinline__ void item_of(const GeoR4& g, int it, int& p, int& c0, int& rb0, int& nu) {
  const int col = it / g.splits, sp = it - col * g.splits;
  p = col / g.ncs;
  c0 = (col - p * g.ncs) * g.wseg;
  rb0 = sp * g.per;
  nu = min(g.per, g.nrb - rb0);
}
__device__ __forceinline__ int rows_lo(int rb0) { return max(0, R * rb0 - 5); }
__device__ __forceinline__ int rows_hi(const GeoR4& g, int rb0, int nu) { return min(g.n1, R * (rb0 + nu) + 5); }
}  // namespace

// Fused metrics (di_recover_metrics): with xtrue != null each epilogue thread also reads the
// ground truth of the outputs it writes and accumulates, in fp64 and a fixed order, sum (x_hat - x)^2, sum x^2 and
// max x; per item, image and warp the sums go to mpart[item][image][warp][3] (no atomics), and k_metrics_finish
// combines the items of each image in item order: PSNR, NMSE and success without a
// second pass over x_hat.
template <bool METRICS>
__global__ void __launch_bounds__(256, 1)
    k_conv3_r4(const __grid_constant__ CUtensorMap tmH2, const uint8_t* __restrict__ tpack,
               const float* __restrict__ bias, int fullmap, int relu, GeoR4 g, float* __restrict__ xhat,
               const float* __restrict__ xtrue, double* __restrict__ mpart) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const int rowb = g.N * 64;                                  // one strip row: 2 images x PP positions x 64 B
  const int chunk_bytes = CHR * rowb;                         // a multiple of 1024 (PP a multiple of 16)
  uint8_t* const tb = smem;                                   // T stack (1024-aligned)
  uint8_t* const ring = smem + TBYTES;                        // NSL chunk slots
  float* const S = reinterpret_cast<float*>(ring + NSL * chunk_bytes);

  __shared__ uint64_t wbar, cfull[NSL], cempty[NSL], acc_full[NACC], acc_empty[NACC];
  __shared__ uint32_t tslot;
  const int warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmH2);
    mbar_init(&wbar, 1);
    for (int s = 0; s < NSL; ++s) mbar_init(&cfull[s], 1), mbar_init(&cempty[s], 1);
    for (int a = 0; a < NACC; ++a) mbar_init(&acc_full[a], 1), mbar_init(&acc_empty[a], 4);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&tslot), tmem_relinquish();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  griddep_wait();                 // the preceding grid's outputs (PDL: only the prologue above overlapped it)
  griddep_launch_dependents();

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ producer: T once, strip chunks
      mbar_arrive_expect_tx(&wbar, TBYTES);
      bulk_load(tb, tpack, TBYTES, &wbar);
      // L2 prefetch cursor, PF chunks ahead of the loads (the ring's lead is too few bytes in flight to cover DRAM
      // latency; the prefetched chunks arrive from L2)
      int pit = blockIdx.x, ps = 0, phi = 0, pp = 0, pc0 = 0;
      auto start_item = [&]() {
        if (pit >= g.items) return;
        int rb0, nu;
        item_of(g, pit, pp, pc0, rb0, nu);
        ps = rows_lo(rb0), phi = rows_hi(g, rb0, nu);
      };
      start_item();
      auto prefetch_next = [&]() {
        if (pit >= g.items) return;
        tma_prefetch_l2_4d(&tmH2, 0, pc0 - 5, 2 * pp, ps);
        if ((ps += CHR) >= phi) pit += gridDim.x, start_item();
      };
      if (C3R_PF > 0)
        for (int i = 0; i < C3R_PF; ++i) prefetch_next();
      uint32_t gc = 0;                 // chunks issued by this CTA
      for (int it = blockIdx.x; it < g.items; it += gridDim.x) {
        int p, c0, rb0, nu;
        item_of(g, it, p, c0, rb0, nu);
        for (int s = rows_lo(rb0), se = rows_hi(g, rb0, nu); s < se; s += CHR, ++gc) {
          const uint32_t sl = gc % NSL;
          if (gc >= NSL) mbar_wait(&cempty[sl], ((gc / NSL) - 1) & 1);
          mbar_arrive_expect_tx(&cfull[sl], chunk_bytes);
          tma_load_4d(ring + sl * chunk_bytes, &tmH2, &cfull[sl], 0, c0 - 5, 2 * p, s);
          if (C3R_PF > 0) prefetch_next();
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
      const uint64_t rstep = (uint64_t)(rowb >> 4);
      constexpr uint64_t TSTEP = TBLK >> 4;                                     // one T entry
      const uint64_t aw0 = adesc0 + (uint64_t)(10 - IMIN) * TSTEP;              // window 0: T[10]
      uint64_t bd = bdesc0;            // ring slot sl of the next row
      uint32_t sl = 0, ph = 0;         // ring slot, its fill parity
      uint32_t an = 0, aph = 0;        // TMEM slot of the next unit to start, and its reuse parity
      int pi = 0;                      // units started (CTA-wide)
#ifdef DI_PROF_CONV3
      long long pc_chunk = 0, pc_acc = 0, pc0 = clock64(), pt;
#define C3P0 pt = clock64();
#define C3P1(acc) acc += clock64() - pt;
#else
#define C3P0
#define C3P1(acc)
#endif
      for (int it = blockIdx.x; it < g.items; it += gridDim.x) {
        int p, c0, rb0, nu;
        item_of(g, it, p, c0, rb0, nu);
        const int slo = rows_lo(rb0), shi = rows_hi(g, rb0, nu);
        uint32_t dold = 0, aold = 0;
        for (int jg = rb0; jg <= rb0 + nu; ++jg) {
          const bool hasN = jg < rb0 + nu, hasO = jg > rb0;
          const int sb = R * jg - 5;                                    // strip row of ka = 0
          const int klo = max(0, slo - sb), khi = min(R, shi - sb);
          // a starting unit has rows in its first group (its accumulate-0 MMA), and N fits one TMEM slot
          DI_DEVICE_ASSERT(!hasN || (klo < khi && klo <= 5), klo, khi);
          DI_DEVICE_ASSERT(g.N <= ACOLS, g.N, ACOLS);
          uint32_t dnew = 0;
          if (hasN) {                                                   // unit jg starts in this group
            if (pi >= NACC) {
              C3P0 mbar_wait(&acc_empty[an], aph ^ 1); C3P1(pc_acc)
              tc_fence_after();
            }
            dnew = tmem + an * ACOLS;
          }
#pragma unroll
          for (int ka = 0; ka < R; ++ka) {
            if (ka < klo || ka >= khi) continue;
            C3P0 mbar_wait(&cfull[sl], ph); C3P1(pc_chunk)
            tc_fence_after();
            if (hasO && ka < NWIN - R) {                                // unit jg - 1, window ka + 11
              const uint64_t ad = aw0 - (uint64_t)(ka + R) * TSTEP;
              umma_f16_ss(dold, ad, bd, idesc, 1);
              umma_f16_ss(dold, ad + 2, bd + 2, idesc, 1);              // channels 16..31: +32 B
            }
            if (hasN) {                                                 // unit jg, window ka
              const uint64_t ad = aw0 - (uint64_t)ka * TSTEP;
              umma_f16_ss(dnew, ad, bd, idesc, ka != klo);
              umma_f16_ss(dnew, ad + 2, bd + 2, idesc, 1);
            }
            umma_commit(&cempty[sl]);                                   // the row is consumed
            bd += rstep;
            if (++sl == NSL) sl = 0, ph ^= 1, bd = bdesc0;
          }
          if (hasO) umma_commit(&acc_full[aold]);                       // unit jg - 1 is complete
          if (hasN) {
            dold = dnew, aold = an;
            ++pi;
            if (++an == NACC) an = 0, aph ^= 1;
          }
        }
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
    // x_hat[row t][j] = sum_v S[t ES + v][j + v] -- 128 threads, consecutive j per warp (conflict-free).  Image i of
    // the pair is TMEM columns i PP .. i PP + 75 of the unit's slot.
    const int q = warp - 4, e = threadIdx.x - 128;
    const float bsc = (!fullmap && bias) ? bias[0] : 0.f;
    int pi = 0;
    for (int it = blockIdx.x; it < g.items; it += gridDim.x) {
      int p, c0, rb0, nu;
      item_of(g, it, p, c0, rb0, nu);
      double m_se[2] = {0.0, 0.0}, m_sx[2] = {0.0, 0.0};
      float m_mx[2] = {-INFINITY, -INFINITY};
      for (int j = rb0; j < rb0 + nu; ++j, ++pi) {
        const int r0 = j * R;
        const int a = pi % NACC;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int b = 2 * p + i;
          // METRICS: the ground truth of this thread's outputs, loaded before the accumulator wait / TMEM load
          float tv[OPT];
          if (METRICS) {
#pragma unroll
            for (int h = 0; h < OPT; ++h) {
              const int idx = e + 128 * h, t = idx >> 6, jc = idx & 63, row = r0 + t;
              tv[h] = (b < g.batch && idx < RP * 64 && jc < g.wseg && c0 + jc < g.n2 && row < g.n1)
                          ? __ldg(xtrue + ((size_t)b * g.n1 + row) * g.n2 + c0 + jc) : 0.f;
            }
          }
          if (i == 0) mbar_wait(&acc_full[a], (pi / NACC) & 1);
          tc_fence_after();
          const uint32_t taddr = tmem + a * ACOLS + i * g.PP + ((uint32_t)(q * 32) << 16);
          uint32_t r[76];             // outputs j < 64 read columns j + v <= 73
          tmem_ld32(taddr, r);
          tmem_ld32(taddr + 32, r + 32);
          tmem_ld8(taddr + 64, r + 64);
          tmem_ld4(taddr + 72, r + 72);
          tmem_ld_wait();
          if (i == 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[a]);
          }
          named_bar(1, 128);          // the previous image's sums are done with S
          const int L = q * 32 + lane;
          if (L < SROWS) {
            float4* dst = reinterpret_cast<float4*>(S + L * SROW);
#pragma unroll
            for (int jj = 0; jj < 19; ++jj)
              dst[jj] = make_float4(__uint_as_float(r[4 * jj]), __uint_as_float(r[4 * jj + 1]),
                                    __uint_as_float(r[4 * jj + 2]), __uint_as_float(r[4 * jj + 3]));
          }
          named_bar(1, 128);          // S holds every tap row of this image and unit
          if (b >= g.batch) continue;
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
                m_se[i] += dd * dd, m_sx[i] += (double)tt * (double)tt, m_mx[i] = fmaxf(m_mx[i], tt);
              }
            }
          }
        }
      }
      if (METRICS) {   // the warp's sums for this item and each image, butterfly order fixed
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          for (int o = 16; o > 0; o >>= 1) {
            m_se[i] += __shfl_xor_sync(0xffffffffu, m_se[i], o);
            m_sx[i] += __shfl_xor_sync(0xffffffffu, m_sx[i], o);
            m_mx[i] = fmaxf(m_mx[i], __shfl_xor_sync(0xffffffffu, m_mx[i], o));
          }
          if (lane == 0) {
            double* mp = mpart + (((size_t)it * 2 + i) * 4 + q) * 3;
            mp[0] = m_se[i], mp[1] = m_sx[i], mp[2] = (double)m_mx[i];
          }
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
  g.n1 = n1, g.n2 = n2, g.batch = batch;
  g.wseg = n2 < 64 ? n2 : 64;
  g.PP = conv3_r4_box_cols(n2);
  g.N = 2 * g.PP;
  g.nrb = (n1 + R - 1) / R;
  g.ncs = (n2 + g.wseg - 1) / g.wseg;
  const int cols = (batch + 1) / 2 * g.ncs;
  // fewer pair-columns than SMs: split each into parts of `per` row blocks
  g.splits = cols >= num_sms ? 1 : std::min(g.nrb, (num_sms + cols - 1) / cols);
  g.per = (g.nrb + g.splits - 1) / g.splits;
  g.splits = (g.nrb + g.per - 1) / g.per;
  g.items = cols * g.splits;
  return g;
}

static size_t smem_r4(int n2) {
  const size_t chunk = (size_t)CHR * 2 * conv3_r4_box_cols(n2) * 64;
  return TBYTES + NSL * chunk + (size_t)SROWS * SROW * 4 + 1024;
}

int conv3_r4_box_rows() { return CHR; }
// positions per image in a strip row: the W + 10 padded columns rounded up to 16 (2 PP = the MMA N, a multiple of 16)
int conv3_r4_box_cols(int n2) { return ((n2 < 64 ? n2 : 64) + 10 + 15) & ~15; }
int conv3_r4_tpack_bytes() { return TBYTES; }

cudaError_t setup_conv3_r4(int n2) {
  const cudaError_t e = cudaFuncSetAttribute(k_conv3_r4<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem_r4(n2));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_conv3_r4<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_r4(n2));
}

// per image b (pair p = b / 2, i = b % 2): the items of pair p (per_pair consecutive items), four warps each, summed
// in that order
__global__ void k_metrics_finish(const double* __restrict__ mpart, int per_pair, int N, int batch,
                                 double* __restrict__ out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  double se = 0.0, sx = 0.0, mx = -INFINITY;
  const int p = b >> 1, i = b & 1;
  for (int t = 0; t < per_pair; ++t) {
    const double* q = mpart + (((size_t)(p * per_pair + t) * 2 + i) * 4) * 3;
    for (int w = 0; w < 4; ++w) se += q[3 * w], sx += q[3 * w + 1], mx = fmax(mx, q[3 * w + 2]);
  }
  const double mse = se / N;
  out[b] = mse == 0.0 ? INFINITY : 10.0 * log10(mx * mx / mse);
  const double nmse = se / sx;
  out[batch + b] = nmse;
  out[2 * batch + b] = nmse <= 0.1 ? 1.0 : 0.0;
}

size_t conv3_r4_metrics_part_bytes(int batch, int n1, int n2, int num_sms) {
  const GeoR4 g = make_geo_r4(batch, n1, n2, num_sms);
  return (size_t)g.items * 2 * 4 * 3 * sizeof(double);
}

cudaError_t launch_conv3_r4(const CUtensorMap* tmH2, const void* tpack, const float* bias, int fullmap, int relu,
                            float* xhat, int batch, int n1, int n2, int num_sms, cudaStream_t st, const float* xtrue,
                            double* mpart, double* metrics) {
  GeoR4 g = make_geo_r4(batch, n1, n2, num_sms);
  const int grid = g.items < num_sms ? g.items : num_sms;
  if (xtrue)
    launch_ex(k_conv3_r4<true>, dim3(grid), dim3(256), smem_r4(n2), st, 1, true, *tmH2,
              reinterpret_cast<const uint8_t*>(tpack), bias, fullmap, relu, g, xhat, xtrue, mpart);
  else
    launch_ex(k_conv3_r4<false>, dim3(grid), dim3(256), smem_r4(n2), st, 1, true, *tmH2,
              reinterpret_cast<const uint8_t*>(tpack), bias, fullmap, relu, g, xhat, (const float*)nullptr,
              (double*)nullptr);
  if (xtrue) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_metrics_finish<<<(batch + 127) / 128, 128, 0, st>>>(mpart, g.ncs * g.splits, n1 * n2, batch, metrics);
  }
  return cudaGetLastError();
}

DI_DEBUG_BINDER(di_debug_bind_k_conv3_r4)

}  // namespace di
