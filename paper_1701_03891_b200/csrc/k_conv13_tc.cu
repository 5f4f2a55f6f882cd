// k_conv13_tc.cu -- the thin conv layers of DeepInverse on the 5th-generation tensor cores (bf16 path):
//   stage 1, conv layer 1: 64 filters 11x11x1  + bias + ReLU, crop S   (Eq. (1))
//   stage 3, conv layer 3:  1 filter  11x11x32 + bias (+ReLU iff DI_FLAG_FINAL_RELU), crop S
// Both are 'same' zero-padded cross-correlations with the flipped taps W' (DESIGN.md §2 Q3).
//
// Common structure (as k_conv2_tc.cu): work unit = (image b, R output rows from r0, <= 64 columns from c0);
// positions are linear in a zero-padded strip of pitch P, so tap (u, v) of output position o reads strip
// position o + u*P + v.  PIXELS ARE THE UMMA N DIMENSION (N = 256 positions per tile) and the weights are the
// A operand of a weight-stationary MMA (tcgen05.mma.ws, M = 32 or 64) -- measured on B200 at the full
// tensor rate for M = 64, N = 256 (tools/ladder.cu t7/t9), where the M = 128 form would waste half the tile.
//
// conv1 (C_in = 1): the K dimension is 16 column taps v of ONE tap row u.  A smem "im2row" buffer holds, for
// every strip position m, the 16 values strip[m .. m+15] (a 32-B row, SWIZZLE_32B), built by two builder
// warps from x_tilde.  K-block u (11 of them) is one MMA whose B operand is the im2row window starting at
// row n0 + u*P (a descriptor address change):  D[f][n] = sum_u sum_v W'[f][u][v] x~[n + u*P + v]  -- every
// output is complete after the 11 MMAs, no epilogue shifts.  M = 64 filters, N = 256 positions.
//
// conv3 (C_out = 1): the K dimension is the 32 input channels (one 64-B NHWC row per position, SWIZZLE_64B,
// strip loaded by one 4-D TMA box with out-of-bounds zero fill = the zero padding of Eq. (1)).  A rows are the
// 11 column taps v of tap row u (M = 32, rows 11..31 zero); K-block u shifts the B window by u*P, so
//   D[v][n] = sum_u sum_c W'[c][u][v] h2[c][n + u*P]   and   x_hat[o] = sum_v D[v][o + v]  (+ bias),
// the last sum (11 lanes at column offsets v) done by the epilogue through shared memory.  A tile of 256
// positions yields 246 complete outputs.
//
// Roles: warp 0 producer (weights once; conv3: TMA strips), warp 1 single-thread MMA issuer, warps 2-3 conv1
// im2row builders (warp 2 also allocates TMEM), epilogue warps 4-7 (conv3) / 4-11 (conv1) on the TMEM quadrants.
// Strips / im2row buffers are double-buffered across units; accumulators rotate over 4 TMEM slots.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "kernels.cuh"
#define DI_TU_ID 2
#include "sm100.cuh"

namespace di {

namespace {
constexpr int NACC = 4;

struct Geo13 {
  int n1, n2, wseg, P, R, nrb, ncs, units, guard;   // guard: finite rows kept past each conv3 strip
};

__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------- conv1 geometry
constexpr int R1 = C1TC_ROWS;           // output rows per unit
constexpr int P1MAX = 80;
constexpr int IM_ROWS = (R1 + 10) * 64;                  // im2row rows per buffer: (R + 10) rows x W <= 64
constexpr int IM_BYTES = IM_ROWS * 32;
constexpr int STRIP_WORDS = ((R1 + 10) * P1MAX + 32) / 2; // strip_lin as words (zero past the real strip)
constexpr int SW1_OFF = ((STRIP_WORDS + 31) & ~31) + 16;  // word offset of the one-element-shifted copy
constexpr int FILL_PER_THREAD = ((R1 + 10) * P1MAX + 63) / 64;   // strip elements per builder thread
constexpr int XC_STRIDE = ((R1 + 10) * (P1MAX + 8) * 2 + 64 + 127) & ~127;   // TMA strip buffer stride (bytes)
constexpr int W1_BYTES = 11 * 64 * 32;                   // 11 tap rows x 64 filters x 16 taps bf16
constexpr int C1_STRIPS = 2 * XC_STRIDE > 2 * SW1_OFF * 4 ? 2 * XC_STRIDE : 2 * SW1_OFF * 4;
constexpr int C1_STAGE_OFF = (W1_BYTES + 2 * IM_BYTES + C1_STRIPS + 1023) & ~1023;
constexpr int C1_STAGE = 4096;                           // one warp's 128 positions x 16 channels of h1, bf16

// ---------------------------------------------------------------- conv3 geometry
constexpr int R3 = C3TC_ROWS;
constexpr int OUT3 = 256 - 10;
constexpr int W3_BYTES = 11 * 32 * 64;                   // 11 tap rows x 32 (v) rows x 32 ch bf16
constexpr int SROW = 267;                                // S row stride (floats), odd -> conflict-free
}  // namespace

// =============================================================================================== conv1
// im2row rows are indexed by OUTPUT position p = r * W + c (W = wseg, no padding positions): row p holds the 16
// values x~[r + u - 5][c - 5 .. c + 10] for the tap row u of the current K-block, i.e. strip[r + u][c .. c + 15] of the
// zero-padded strip (pitch P); K-block u reads the window starting at row p0 + u * W.  A tile is 256 consecutive
// output positions, so its outputs are contiguous in NHWC h1 whenever the unit spans the full image width.
// Epilogue: tcgen05.ld.16x256b gives thread t the TMEM lanes t/4 and t/4 + 8 of a 16-lane group at columns
// 2(t%4), 2(t%4)+1 (tools/ladder.cu t15) -- the fragment layout of stmatrix, whose .trans form writes the NHWC
// transpose into a per-warp staging buffer that one TMA tensor store per half tile moves to h1.
// TMAX = true (n2 % 8 == 0): the strip arrives by TMA (out-of-bounds zero fill), double-buffered across units and
// issued one unit ahead; TMAX = false: builders gather it with plain loads (any n2).  (A TMA box whose innermost
// start coordinate is not 16-B aligned faults on B200 -- tools/scratch/tma3d.cu -- hence the 8-column left margin.)
template <bool TMAX>
__global__ void __launch_bounds__(384, 1)
    k_conv1_tc(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmS, int tma_store,
               const __nv_bfloat16* __restrict__ xt, const uint8_t* __restrict__ w1pack, const float* __restrict__ bias,
               int fullmap, Geo13 g, __nv_bfloat16* __restrict__ h1) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* wbuf = smem;                                           // 22 KB
  uint8_t* const im0 = smem + W1_BYTES;   // 2 im2row buffers (1024-aligned: W1_BYTES = 22528)
  uint32_t* const sw0 = reinterpret_cast<uint32_t*>(smem + W1_BYTES + 2 * IM_BYTES);
  uint32_t* const sw1 = sw0 + SW1_OFF;
  uint8_t* const xc0 = smem + W1_BYTES + 2 * IM_BYTES;   // TMAX: 2 buffers x 8 shifted copies (aliases sw0/sw1)
  uint8_t* const stage0 = smem + C1_STAGE_OFF;              // epilogue: 8 warps x 2 x 4 KB h1 staging (SWIZZLE_32B)

  __shared__ uint64_t wbar, im_full[2], im_empty[2], acc_full[NACC], acc_empty[NACC], xfull[2];
  __shared__ uint32_t tslot;
  const int warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    mbar_init(&wbar, 1);
    for (int s = 0; s < 2; ++s) mbar_init(&im_full[s], 64), mbar_init(&im_empty[s], 1);
    for (int a = 0; a < NACC; ++a) mbar_init(&acc_full[a], 1), mbar_init(&acc_empty[a], 8);
    for (int s = 0; s < 2; ++s) mbar_init(&xfull[s], 1);
    if (TMAX) tma_prefetch_desc(&tmX);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&tslot), tmem_relinquish();
  if (TMAX) {   // zero the tails past each copy (TMA never writes them; windows of the last rows read them)
    for (int i = threadIdx.x; i < 2 * XC_STRIDE / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(xc0)[i] = 0u;
    fence_async_smem();
  } else {
    for (int i = threadIdx.x; i < 2 * SW1_OFF; i += blockDim.x) sw0[i] = 0u;   // zero tails of both copies
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  griddep_wait();                 // the preceding grid's outputs (PDL: only the prologue above overlapped it)
  griddep_launch_dependents();
  const int per_img = g.nrb * g.ncs;
  const int P = g.P, W = g.wseg;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ weights, once
      mbar_arrive_expect_tx(&wbar, W1_BYTES);
      bulk_load(wbuf, w1pack, W1_BYTES, &wbar);
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      mbar_wait(&wbar, 0);
      tc_fence_after();
      const uint64_t adesc0 = smem_desc(smem_u32(wbuf), 16, 256, kSwizzle32B);
      const uint64_t bdesc_base = smem_desc(smem_u32(im0), 16, 256, kSwizzle32B);
      const uint64_t bstep = (uint64_t)((W * 32) >> 4);
      int it = 0, ti = 0;
#ifdef DI_PROF_CONV1
      long long c_im = 0, c_acc = 0, c0_ = clock64();
#endif
      for (int u = blockIdx.x; u < g.units; u += gridDim.x, ++it) {
        const int rem = u % per_img;
        const int r0 = (rem / g.ncs) * g.R;
        const int npos = min(g.R, g.n1 - r0) * W;
        const int s = it & 1;
#ifdef DI_PROF_CONV1
        long long t0 = clock64();
#endif
        mbar_wait(&im_full[s], (it >> 1) & 1);
#ifdef DI_PROF_CONV1
        c_im += clock64() - t0;
#endif
        tc_fence_after();
        for (int n0 = 0; n0 < npos; n0 += 256, ++ti) {
          const int cnt = min(256, npos - n0);
          const int N = cnt > 128 ? 256 : (cnt > 64 ? 128 : 64);
          const uint32_t idesc = idesc_f32acc(1, 64, N);
          const int a = ti % NACC;
#ifdef DI_PROF_CONV1
          long long t1 = clock64();
#endif
          if (ti >= NACC) mbar_wait(&acc_empty[a], ((ti / NACC) - 1) & 1);
#ifdef DI_PROF_CONV1
          c_acc += clock64() - t1;
#endif
          tc_fence_after();
          const uint32_t d = tmem + a * 128;
          DI_DEVICE_ASSERT(n0 + 10 * W + N <= IM_ROWS, n0, N);   // the u = 10 window stays in the im2row buffer
          uint64_t bd = bdesc_base + (uint64_t)(((s * IM_BYTES) + n0 * 32) >> 4);
#pragma unroll
          for (int tu = 0; tu < 11; ++tu) {
            umma_ws_f16(d, adesc0 + (uint64_t)((tu * 2048) >> 4), bd, idesc, tu != 0);
            bd += bstep;
          }
          umma_commit(&acc_full[a]);
        }
        umma_commit(&im_empty[s]);
      }
#ifdef DI_PROF_CONV1
      if (blockIdx.x % 37 == 0)
        printf("conv1 cta %d issuer: cycles %lld im-wait %lld acc-wait %lld units %d tiles %d\n", blockIdx.x,
               clock64() - c0_, c_im, c_acc, it, ti);
#endif
    }
  } else if (warp < 4) {  // ------------------------------------------- im2row builders (64 threads)
    // strip_lin[idx] = x_tilde[b][r0-5+rr][c0-5+cc] (zero outside the image and past the 5-px halo), kept twice
    // as 32-bit words: sw0 = strip_lin, sw1 = strip_lin shifted by one element, so that the 16-element window
    // starting at ANY strip position m is 8 aligned words (from sw0 if m is even, sw1 if odd).  sw1 sits 16 words
    // (mod 32) after sw0: a warp's 32 consecutive rows read 32 distinct banks.
    const int bt = threadIdx.x - 64;
    uint16_t* s0 = reinterpret_cast<uint16_t*>(sw0);
    uint16_t* s1 = reinterpret_cast<uint16_t*>(sw1);
    const uint32_t wmagic = (1u << 20) / (uint32_t)W + 1;   // p / W for p < 2^13 (W <= 64)
    int it = 0;
#ifdef DI_PROF_CONV1
    long long b_wait = 0, b_load = 0, b_build = 0, b0_ = clock64();
#endif
    for (int u = blockIdx.x; u < g.units; u += gridDim.x, ++it) {
      const int b = u / per_img, rem = u - b * per_img;
      const int r0 = (rem / g.ncs) * g.R, c0 = (rem % g.ncs) * g.wseg;
      const int s = it & 1;
#ifdef DI_PROF_CONV1
      long long bt0 = clock64();
#endif
      if (it >= 2) mbar_wait(&im_empty[s], ((it >> 1) - 1) & 1);
#ifdef DI_PROF_CONV1
      long long bt1 = clock64();
      b_wait += bt1 - bt0;
#endif
      uint8_t* dst = im0 + s * IM_BYTES;
      const int nrows = (g.R + 10) * W;
#ifdef DI_PROF_CONV1
      long long bt2 = 0;
#endif
      if (TMAX) {
        if (bt == 0) {
          // the strip of unit `un` into buffer `buf` (unit it+1 is issued one unit ahead).  TMA needs a 16-B
          // aligned innermost start, so the box starts 8 columns left of the unit (not 5): strip[r][cc] sits at
          // copy[r * Q + cc + 3] with Q = P + 8.
          for (int k = (it == 0 ? 0 : 1); k < 2; ++k) {
            const int un = u + k * gridDim.x, buf = (it + k) & 1;
            if (un >= g.units) break;
            const int bb = un / per_img, rm = un - bb * per_img;
            const int rr0 = (rm / g.ncs) * g.R, cc0 = (rm % g.ncs) * g.wseg;
            mbar_arrive_expect_tx(&xfull[buf], (g.R + 10) * (P + 8) * 2);
            tma_load_3d(xc0 + buf * XC_STRIDE, &tmX, &xfull[buf], cc0 - 8, rr0 - 5, bb);
          }
        }
        mbar_wait(&xfull[s], (it >> 1) & 1);
#ifdef DI_PROF_CONV1
        bt2 = clock64();
        b_load += bt2 - bt1;
#endif
        // row p -> copy position m = r*Q + c + 3; its 16-element window = 8 words funnel-shifted by (m & 1) * 16
        const uint32_t* xw = reinterpret_cast<const uint32_t*>(xc0 + s * XC_STRIDE);
        const int Q = P + 8;
        for (int p = bt; p < nrows; p += 64) {
          const int r = (int)(((uint32_t)p * wmagic) >> 20), c = p - r * W;
          const int m = r * Q + c + 3;
          const uint32_t* w = xw + (m >> 1);
          const uint32_t sh = (m & 1) * 16;
          uint32_t o[8];
          uint32_t prev = w[0];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint32_t nxt = w[i + 1];
            o[i] = __funnelshift_r(prev, nxt, sh);
            prev = nxt;
          }
          const int sw = (p >> 2) & 1;
          *reinterpret_cast<uint4*>(dst + p * 32 + (sw << 4)) = make_uint4(o[0], o[1], o[2], o[3]);
          *reinterpret_cast<uint4*>(dst + p * 32 + ((1 ^ sw) << 4)) = make_uint4(o[4], o[5], o[6], o[7]);
        }
      } else {
        const uint16_t* src = reinterpret_cast<const uint16_t*>(xt) + (size_t)b * g.n1 * g.n2;
        // all loads of this thread first (memory-level parallelism), then the shared-memory stores
        const int strip_real = (g.R + 10) * P;
        uint16_t v[FILL_PER_THREAD];
  #pragma unroll
        for (int i = 0; i < FILL_PER_THREAD; ++i) {
          const int idx = bt + 64 * i;
          const int rr = idx / P, cc = idx - rr * P;
          const int gy = r0 - 5 + rr, gx = c0 - 5 + cc;
          v[i] = 0;
          if (idx < strip_real && cc < g.wseg + 10 && gy >= 0 && gy < g.n1 && gx >= 0 && gx < g.n2)
            v[i] = src[(size_t)gy * g.n2 + gx];
        }
  #pragma unroll
        for (int i = 0; i < FILL_PER_THREAD; ++i) {
          const int idx = bt + 64 * i;
          if (idx < strip_real) {
            s0[idx] = v[i];
            if (idx > 0) s1[idx - 1] = v[i];
          }
        }
        named_bar(2, 64);
  #ifdef DI_PROF_CONV1
        bt2 = clock64();
        b_load += bt2 - bt1;
  #endif
        // im2row row p (output position r*W + c) = strip_lin[r*P + c .. +15], SWIZZLE_32B
        // (16-B chunk h of row p at p*32 + ((h ^ (p>>2 & 1)) << 4))
        for (int p = bt; p < nrows; p += 64) {
          const int r = (int)(((uint32_t)p * wmagic) >> 20), c = p - r * W;
          const int m = r * P + c;
          const uint32_t* w = ((m & 1) ? sw1 : sw0) + (m >> 1);
          const int sw = (p >> 2) & 1;
          *reinterpret_cast<uint4*>(dst + p * 32 + (sw << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
          *reinterpret_cast<uint4*>(dst + p * 32 + ((1 ^ sw) << 4)) = make_uint4(w[4], w[5], w[6], w[7]);
        }
      }
      fence_async_smem();
      mbar_arrive(&im_full[s]);
      named_bar(2, 64);  // the strip is refilled for the next unit only after every builder is done reading it
#ifdef DI_PROF_CONV1
      b_build += clock64() - bt2;
#endif
    }
#ifdef DI_PROF_CONV1
    if (blockIdx.x % 37 == 0 && bt == 0)
      printf("conv1 cta %d builder: cycles %lld wait %lld strip-load %lld im2row %lld\n", blockIdx.x,
             clock64() - b0_, b_wait, b_load, b_build);
#endif
  } else {  // -------------------------------------------------------- epilogue, warps 4..11
    // .ws M=64 D layout: quadrants {0,1} = filter rows 0..63 for tile columns [0, N/2), {2,3} for [N/2, N).
    // Warp w reads quadrant q = w % 4, 16-lane group hh = (w - 4) / 4 = channels 16G .. 16G + 15, G = 2(q&1) + hh
    // (packed filter rows in natural order).  tcgen05.ld.16x256b gives thread t channels ca = 16G + t/4 and
    // cb = ca + 8 at columns 2(t%4), 2(t%4)+1 of each 8-column block k: with bias + ReLU and bf16 rounding these are
    // the fragments of two 8 x 8 [channel][position] matrices per block, and stmatrix.trans writes their transposes
    // -- [position][8 channels], i.e. NHWC -- into the warp's staging buffer (32-B rows = 16 channels, SWIZZLE_32B).
    // A full 128-position half tile (two 64-column image rows) then leaves by ONE TMA tensor store per warp
    // (box 16 ch x 64 cols x 2 rows, out-of-range rows clipped by the TMA unit): full-sector writes and no per-lane
    // store instructions.  Other tiles (narrow images, ragged tiles, full-map biases) copy rows out with 16-B stores.
    const int q = warp & 3, hh = (warp - 4) >> 2;
    const int i4 = lane >> 2, cpair = 2 * (lane & 3);
    const int G = 2 * (q & 1) + hh;
    const int ca = 16 * G + i4, cb = ca + 8;                  // this thread's channels
    const float ba = (!fullmap && bias) ? bias[ca] : 0.f, bb = (!fullmap && bias) ? bias[cb] : 0.f;
    const uint32_t wmagic = (1u << 20) / (uint32_t)W + 1;
    uint8_t* const stg = stage0 + (warp - 4) * 2 * C1_STAGE;
    int ti = 0, sb = 0;
    for (int u = blockIdx.x; u < g.units; u += gridDim.x) {
      const int b = u / per_img, rem = u - b * per_img;
      const int r0 = (rem / g.ncs) * g.R, c0 = (rem % g.ncs) * g.wseg;
      const int npos = min(g.R, g.n1 - r0) * W;
      const bool linear = g.ncs == 1;    // the unit spans the full width: outputs are contiguous in h1
      const size_t pix0 = ((size_t)b * g.n1 + r0) * g.n2 + c0;
      for (int n0 = 0; n0 < npos; n0 += 256, ++ti) {
        const int cnt = min(256, npos - n0);
        const int N = cnt > 128 ? 256 : (cnt > 64 ? 128 : 64);
        const int half = N / 2;
        const int a = ti % NACC;
        mbar_wait(&acc_full[a], (ti / NACC) & 1);
        tc_fence_after();
        const int pbase = n0 + (q >> 1) * half;
        const uint32_t taddr = tmem + a * 128 + ((uint32_t)(q * 32 + 16 * hh) << 16);
        const bool tma = tma_store && N == 256 && W == 64 && !fullmap;
        uint8_t* const buf = stg + sb * C1_STAGE;
        if (lane == 0) bulk_wait_read<1>();   // this buffer's previous store (two half tiles ago) has read it
        __syncwarp();
        const uint32_t sbase = smem_u32(buf);
        for (int c = 0; c < half; c += 32) {
          uint32_t r[16];
          tmem_ld_16x256b_x4(taddr + c, r);
          tmem_ld_wait();
          uint32_t f[8];   // f[2k] = channels ca.. of block k, f[2k + 1] = channels cb.. (positions 2(t%4), +1)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            float v[4] = {__uint_as_float(r[4 * k]), __uint_as_float(r[4 * k + 1]), __uint_as_float(r[4 * k + 2]),
                          __uint_as_float(r[4 * k + 3])};
            if (fullmap && bias) {
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int p = min(pbase + c + 8 * k + cpair + e, npos - 1);
                const int rr = (int)(((uint32_t)p * wmagic) >> 20), cc = p - rr * W;
                const size_t pm = ((size_t)(r0 + rr) * g.n2 + min(c0 + cc, g.n2 - 1));
                v[e] += bias[pm * 64 + ca], v[2 + e] += bias[pm * 64 + cb];
              }
            } else {
              v[0] += ba, v[1] += ba, v[2] += bb, v[3] += bb;
            }
            f[2 * k] = pack_bf16x2(fmaxf(v[0], 0.f), fmaxf(v[1], 0.f));
            f[2 * k + 1] = pack_bf16x2(fmaxf(v[2], 0.f), fmaxf(v[3], 0.f));
          }
          // stored matrix j of call h: block k = 2h + j / 2, channel half j % 2; lane 8j + i -> position 8k + i
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int j = lane >> 3, pos = c + 8 * (2 * h + (j >> 1)) + (lane & 7), ch = j & 1;
            stmatrix_x4_trans(sbase + pos * 32 + ((ch ^ ((pos >> 2) & 1)) << 4), f[4 * h], f[4 * h + 1],
                              f[4 * h + 2], f[4 * h + 3]);
          }
        }
        if (tma) {
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_4d(&tmS, buf, 16 * G, c0, r0 + pbase / 64, b);
            bulk_commit_group();
          }
        } else {
          __syncwarp();
          // rows of this half tile: lane -> (position, 16-B channel chunk)
          for (int e = lane; e < 2 * half; e += 32) {
            const int pos = e >> 1, ch = e & 1, p = pbase + pos;
            if (p >= n0 + cnt) continue;
            size_t pix;
            if (linear) {
              pix = pix0 + p;
            } else {
              const int rr = (int)(((uint32_t)p * wmagic) >> 20), cc = p - rr * W;
              if (c0 + cc >= g.n2) continue;
              pix = pix0 + (size_t)rr * g.n2 + cc;
            }
            const uint4 val = *reinterpret_cast<const uint4*>(buf + pos * 32 + ((ch ^ ((pos >> 2) & 1)) << 4));
            *reinterpret_cast<uint4*>(h1 + pix * 64 + 16 * G + 8 * ch) = val;
          }
        }
        sb ^= 1;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[a]);
      }
    }
    if (lane == 0) bulk_wait<0>();   // every h1 store has completed before the CTA exits
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}


// =============================================================================================== conv1, TF32
// TF32 mode (fp32 x_tilde, TF32 products): the same mapping as k_conv1_tc with 64-B im2row rows (16 fp32 taps,
// SWIZZLE_64B, two kind::tf32 K = 8 MMAs per tap row), R = 8 rows per unit, the strip always by TMA (needs
// n2 % 4 == 0; otherwise the SIMT conv1 runs), fp32 h1 stores of channel pairs.
constexpr int R1T = 8;
constexpr int IM_ROWS_T = (R1T + 10) * 64;
constexpr int IM_BYTES_T = IM_ROWS_T * 64;
constexpr int W1T_BYTES = 11 * 64 * 64;                      // 11 tap rows x 64 filters x 16 fp32 taps
constexpr int XT_STRIDE = ((R1T + 10) * (P1MAX + 8) * 4 + 128 + 127) & ~127;

// DG3 = true: the training step's layer-3 data gradient on the same machinery:
//   dH2[p][ci] = [h2[p][ci] > 0] * sum_{u,v} wx3[0][ci][10-u][10-v] * dG3[p + (u-5, v-5)]
// is a 1 -> 32 'same' correlation: the strip is dG3 (tmX over dG3), the packed filters are the rotated layer-3
// taps in rows 0..31 (rows 32..63 zero), and the epilogue writes 32 channels masked by h2 instead of bias+ReLU.
// COUT = 32 (bank rows 32..63 zero) or 64 output channels; DG3 = masked epilogue (no bias / ReLU).
template <int COUT, bool DG3>
__global__ void __launch_bounds__(384, 1)
    k_conv1_tf32(const __grid_constant__ CUtensorMap tmX, const uint8_t* __restrict__ w1pack,
                 const float* __restrict__ bias, int fullmap, Geo13 g, float* __restrict__ h1,
                 const void* __restrict__ mask, int mask_bf16, float* __restrict__ part_b) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  uint8_t* wbuf = smem;                                 // 44 KB
  uint8_t* const im0 = smem + W1T_BYTES;                // 2 im2row buffers
  uint8_t* const xc0 = smem + W1T_BYTES + 2 * IM_BYTES_T;   // 2 strip buffers

  __shared__ uint64_t wbar, im_full[2], im_empty[2], acc_full[NACC], acc_empty[NACC], xfull[2];
  __shared__ uint32_t tslot;
  const int warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    mbar_init(&wbar, 1);
    for (int s = 0; s < 2; ++s) mbar_init(&im_full[s], 64), mbar_init(&im_empty[s], 1), mbar_init(&xfull[s], 1);
    for (int a = 0; a < NACC; ++a) mbar_init(&acc_full[a], 1), mbar_init(&acc_empty[a], 8);
    tma_prefetch_desc(&tmX);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&tslot), tmem_relinquish();
  for (int i = threadIdx.x; i < 2 * XT_STRIDE / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(xc0)[i] = 0u;
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int per_img = g.nrb * g.ncs;
  const int P = g.P, W = g.wseg, Q = P + 8;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ weights, once
      mbar_arrive_expect_tx(&wbar, W1T_BYTES);
      bulk_load(wbuf, w1pack, W1T_BYTES, &wbar);
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      mbar_wait(&wbar, 0);
      tc_fence_after();
      const uint64_t adesc0 = smem_desc(smem_u32(wbuf), 16, 512, kSwizzle64B);
      const uint64_t bdesc_base = smem_desc(smem_u32(im0), 16, 512, kSwizzle64B);
      const uint64_t bstep = (uint64_t)((W * 64) >> 4);
      int it = 0, ti = 0;
      for (int u = blockIdx.x; u < g.units; u += gridDim.x, ++it) {
        const int rem = u % per_img;
        const int r0 = (rem / g.ncs) * g.R;
        const int npos = min(g.R, g.n1 - r0) * W;
        const int s = it & 1;
        mbar_wait(&im_full[s], (it >> 1) & 1);
        tc_fence_after();
        for (int n0 = 0; n0 < npos; n0 += 256, ++ti) {
          const int cnt = min(256, npos - n0);
          const int N = cnt > 128 ? 256 : (cnt > 64 ? 128 : 64);
          const uint32_t idesc = idesc_f32acc(2, DG3 ? 32 : 64, N);   // DG3: 32 bank rows, .ws M = 32
          const int a = ti % NACC;
          if (ti >= NACC) mbar_wait(&acc_empty[a], ((ti / NACC) - 1) & 1);
          tc_fence_after();
          const uint32_t d = tmem + a * 128;
          uint64_t bd = bdesc_base + (uint64_t)(((s * IM_BYTES_T) + n0 * 64) >> 4);
#pragma unroll
          for (int tu = 0; tu < 11; ++tu) {
            const uint64_t ad = adesc0 + (uint64_t)((tu * 4096) >> 4);
            umma_ws_tf32(d, ad, bd, idesc, tu != 0);
            umma_ws_tf32(d, ad + 2, bd + 2, idesc, 1);        // taps 8..15: +32 B
            bd += bstep;
          }
          umma_commit(&acc_full[a]);
        }
        umma_commit(&im_empty[s]);
      }
    }
  } else if (warp < 4) {  // ------------------------------------------- im2row builders (64 threads)
    const int bt = threadIdx.x - 64;
    const uint32_t wmagic = (1u << 20) / (uint32_t)W + 1;
    int it = 0;
    for (int u = blockIdx.x; u < g.units; u += gridDim.x, ++it) {
      const int s = it & 1;
      if (it >= 2) mbar_wait(&im_empty[s], ((it >> 1) - 1) & 1);
      if (bt == 0) {   // strip of unit `un` into buffer `buf`, one unit ahead; box starts 8 columns left (16-B rule)
        for (int k = (it == 0 ? 0 : 1); k < 2; ++k) {
          const int un = u + k * gridDim.x, buf = (it + k) & 1;
          if (un >= g.units) break;
          const int bb = un / per_img, rm = un - bb * per_img;
          const int rr0 = (rm / g.ncs) * g.R, cc0 = (rm % g.ncs) * g.wseg;
          mbar_arrive_expect_tx(&xfull[buf], (g.R + 10) * Q * 4);
          tma_load_3d(xc0 + buf * XT_STRIDE, &tmX, &xfull[buf], cc0 - 8, rr0 - 5, bb);
        }
      }
      mbar_wait(&xfull[s], (it >> 1) & 1);
      // im2row row p (output position r*W + c) = strip[r][c .. c+15] = copy[r*Q + c + 3 ..]; SWIZZLE_64B:
      // 16-B chunk j of row p at p*64 + ((j ^ ((p >> 1) & 3)) << 4)
      const uint32_t* xw = reinterpret_cast<const uint32_t*>(xc0 + s * XT_STRIDE);
      uint8_t* dst = im0 + s * IM_BYTES_T;
      const int nrows = (g.R + 10) * W;
      for (int p = bt; p < nrows; p += 64) {
        const int r = (int)(((uint32_t)p * wmagic) >> 20), c = p - r * W;
        const uint32_t* w = xw + r * Q + c + 3;
        const int sw = (p >> 1) & 3;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          *reinterpret_cast<uint4*>(dst + p * 64 + ((j ^ sw) << 4)) =
              make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
      }
      fence_async_smem();
      mbar_arrive(&im_full[s]);
      named_bar(2, 64);
    }
  } else {  // -------------------------------------------------------- epilogue, warps 4..11 (as k_conv1_tc)
    const int q = warp & 3, hh = (warp - 4) >> 2;
    const int i4 = lane >> 2, cpair = 2 * (lane & 3);
    const int ch = 16 * (2 * (q & 1) + hh) + 2 * i4;
    const float b0 = (!fullmap && bias && ch < COUT) ? bias[ch] : 0.f;
    const float b1 = (!fullmap && bias && ch < COUT) ? bias[ch + 1] : 0.f;
    const uint32_t wmagic = (1u << 20) / (uint32_t)W + 1;
    // DG3: .ws M = 32 puts D columns [qN/4, (q+1)N/4) in lane quadrant q, so all 8 warps hold channels
    // 16 hh + 2 i4 (+1) of their quadrant's positions; the layer-2 bias gradient (sum of dG2) is summed per thread
    const int ch3 = 16 * hh + 2 * i4;
    float bs0 = 0.f, bs1 = 0.f;
    int ti = 0;
    for (int u = blockIdx.x; u < g.units; u += gridDim.x) {
      const int b = u / per_img, rem = u - b * per_img;
      const int r0 = (rem / g.ncs) * g.R, c0 = (rem % g.ncs) * g.wseg;
      const int npos = min(g.R, g.n1 - r0) * W;
      const bool linear = g.ncs == 1;
      const size_t pix0 = ((size_t)b * g.n1 + r0) * g.n2 + c0;
      for (int n0 = 0; n0 < npos; n0 += 256, ++ti) {
        const int cnt = min(256, npos - n0);
        const int N = cnt > 128 ? 256 : (cnt > 64 ? 128 : 64);
        const int half = N / 2;
        const int a = ti % NACC;
        mbar_wait(&acc_full[a], (ti / NACC) & 1);
        tc_fence_after();
        if (DG3) {
          const int quarter = N / 4;
          const int pbq = n0 + q * quarter;
          const uint32_t taddr3 = tmem + a * 128 + ((uint32_t)(q * 32 + 16 * hh) << 16);
          for (int c = 0; c < quarter; c += 32) {
            uint32_t r[16];
            tmem_ld_16x256b_x4(taddr3 + c, r);
            tmem_ld_wait();
            size_t pixv[8];
            bool ok[8];
            float2 m[8];
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {   // all 8 mask loads in flight before the stores
              const int j = c + 8 * (kk >> 1) + cpair + (kk & 1);
              const int p = pbq + j;
              ok[kk] = j < quarter && p < n0 + cnt;
              if (linear) {
                pixv[kk] = pix0 + p;
              } else {
                const int rr = (int)(((uint32_t)p * wmagic) >> 20), cc = p - rr * W;
                ok[kk] = ok[kk] && c0 + cc < g.n2;
                pixv[kk] = pix0 + (size_t)rr * g.n2 + cc;
              }
            }
            if (mask_bf16) {   // BF16 contexts: h2 is bf16 (branch hoisted so the 8 loads issue back to back)
              uint32_t mb[8];
#pragma unroll
              for (int kk = 0; kk < 8; ++kk)
                mb[kk] = ok[kk] ? __ldg(reinterpret_cast<const uint32_t*>(reinterpret_cast<const __nv_bfloat16*>(mask) +
                                                                         pixv[kk] * 32 + ch3))
                                : 0u;
#pragma unroll
              for (int kk = 0; kk < 8; ++kk)
                m[kk] = make_float2(__uint_as_float(mb[kk] << 16), __uint_as_float(mb[kk] & 0xffff0000u));
            } else {
#pragma unroll
              for (int kk = 0; kk < 8; ++kk)
                m[kk] = ok[kk] ? __ldg(reinterpret_cast<const float2*>(reinterpret_cast<const float*>(mask) +
                                                                       pixv[kk] * 32 + ch3))
                               : make_float2(0.f, 0.f);
            }
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {   // dG2 = [h2 > 0] dH2 in bf16 (the dgrad2 / wgrad2 operand)
              const float v0 = m[kk].x > 0.f ? __uint_as_float(r[4 * (kk >> 1) + (kk & 1)]) : 0.f;
              const float v1 = m[kk].y > 0.f ? __uint_as_float(r[4 * (kk >> 1) + 2 + (kk & 1)]) : 0.f;
              if (ok[kk]) {
                bs0 += v0, bs1 += v1;
                *reinterpret_cast<uint32_t*>(reinterpret_cast<__nv_bfloat16*>(h1) + pixv[kk] * 32 + ch3) =
                    pack_bf16x2(v0, v1);
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[a]);
          continue;
        }
        const int pbase = n0 + (q >> 1) * half;
        const uint32_t taddr = tmem + a * 128 + ((uint32_t)(q * 32 + 16 * hh) << 16);
        for (int c = 0; c < half && ch < COUT; c += 32) {   // warps of bank rows >= COUT idle
          uint32_t r[16];
          tmem_ld_16x256b_x4(taddr + c, r);
          tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int p = pbase + c + 8 * k + cpair + e;
              if (p >= n0 + cnt) continue;
              size_t pix;
              if (linear) {
                pix = pix0 + p;
              } else {
                const int rr = (int)(((uint32_t)p * wmagic) >> 20), cc = p - rr * W;
                if (c0 + cc >= g.n2) continue;
                pix = pix0 + (size_t)rr * g.n2 + cc;
              }
              float v0 = __uint_as_float(r[4 * k + e]), v1 = __uint_as_float(r[4 * k + 2 + e]);
              if (fullmap && bias) {
                const size_t pm = pix % ((size_t)g.n1 * g.n2);
                v0 += bias[pm * COUT + ch], v1 += bias[pm * COUT + ch + 1];
              } else {
                v0 += b0, v1 += b1;
              }
              *reinterpret_cast<float2*>(h1 + pix * COUT + ch) = make_float2(fmaxf(v0, 0.f), fmaxf(v1, 0.f));
            }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[a]);
      }
    }
    if (DG3) {   // per-CTA layer-2 bias partials: channel j = sum over its 16 threads in a fixed order
      __shared__ float sb[256][2];
      const int e = threadIdx.x - 128;
      sb[e][0] = bs0, sb[e][1] = bs1;
      named_bar(3, 256);
      if (e < 32) {
        const int h = e >> 4, i = (e & 15) >> 1, w01 = e & 1;
        float t = 0.f;
        for (int qq = 0; qq < 4; ++qq)
          for (int l4 = 0; l4 < 4; ++l4) t += sb[(h * 4 + qq) * 32 + i * 4 + l4][w01];
        part_b[(size_t)blockIdx.x * 32 + e] = t;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// =============================================================================================== conv3
// TF32 = true: fp32 h2 with TF32 products.  An fp32 position row of 32 channels is 128 B, so the channels split into
// two halves of 16 (64-B rows, the bf16 layout); the strip is loaded once per half (strip sequence sk = unit*2 + h,
// double-buffered) and the K-loop runs half-major over the unit's (<= 2) tiles, whose accumulators stay live across
// both halves.  BF16: one "half" of 32 channels.
template <bool TF32>
__global__ void __launch_bounds__(256, 1)
    k_conv3_tc(const __grid_constant__ CUtensorMap tmH2, const uint8_t* __restrict__ w3pack,
               const float* __restrict__ bias, int fullmap, int relu, Geo13 g, float* __restrict__ xhat) {
  constexpr int NH = TF32 ? 2 : 1;
  constexpr int WB = NH * W3_BYTES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const int P = g.P;
  const int strip_bytes = (g.R + 10) * P * 64;
  const int strip_alloc = (strip_bytes + g.guard * 64 + 1023) & ~1023;
  uint8_t* wbuf = smem;                                       // NH x 22 KB (1024-aligned)
  uint8_t* const strip0 = smem + WB;  // 2 strip buffers, strip_alloc apart
  float* S = reinterpret_cast<float*>(smem + WB + 2 * strip_alloc);   // [11][SROW]

  __shared__ uint64_t wbar, sfull[2], sempty[2], acc_full[NACC], acc_empty[NACC];
  __shared__ uint32_t tslot;
  const int warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmH2);
    mbar_init(&wbar, 1);
    for (int s = 0; s < 2; ++s) mbar_init(&sfull[s], 1), mbar_init(&sempty[s], 1);
    for (int a = 0; a < NACC; ++a) mbar_init(&acc_full[a], 1), mbar_init(&acc_empty[a], 4);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<256>(&tslot), tmem_relinquish();
  // Guard rows after each strip: the B windows of the last tile of a unit read up to g.guard rows past the
  // TMA box (their outputs are discarded), but 0 * NaN would not be: keep them finite.
  for (int s = 0; s < 2; ++s)
    for (int i = threadIdx.x; i < g.guard * 64 / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(strip0 + s * strip_alloc + strip_bytes)[i] = make_uint4(0, 0, 0, 0);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int per_img = g.nrb * g.ncs;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ producer
      mbar_arrive_expect_tx(&wbar, WB);
      bulk_load(wbuf, w3pack, WB, &wbar);
      int sk = 0;
      for (int u = blockIdx.x; u < g.units; u += gridDim.x) {
        const int b = u / per_img, rem = u - b * per_img;
        const int r0 = (rem / g.ncs) * g.R, c0 = (rem % g.ncs) * g.wseg;
        for (int h = 0; h < NH; ++h, ++sk) {
          const int s = sk & 1;
          if (sk >= 2) mbar_wait(&sempty[s], ((sk >> 1) - 1) & 1);
          mbar_arrive_expect_tx(&sfull[s], strip_bytes);
          tma_load_4d(strip0 + s * strip_alloc, &tmH2, &sfull[s], 16 * h, c0 - 5, r0 - 5, b);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      mbar_wait(&wbar, 0);
      tc_fence_after();
      constexpr uint32_t idesc = idesc_f32acc(TF32 ? 2 : 1, 32, 256);
      const uint64_t adesc0 = smem_desc(smem_u32(wbuf), 16, 512, kSwizzle64B);
      const uint64_t bdesc_base = smem_desc(smem_u32(strip0), 16, 512, kSwizzle64B);
      const uint64_t bstep = (uint64_t)((P * 64) >> 4);
      int sk = 0, ti = 0;
#ifdef DI_PROF_CONV3
      long long c_s = 0, c_a = 0, c0_ = clock64();
      int it = 0;
#endif
      for (int u = blockIdx.x; u < g.units; u += gridDim.x) {
        const int rem = u % per_img;
        const int r0 = (rem / g.ncs) * g.R;
        const int rows = min(g.R, g.n1 - r0);
        const int L = (rows - 1) * P + g.wseg;
        const int ntiles = (L + OUT3 - 1) / OUT3;
        for (int h = 0; h < NH; ++h, ++sk) {
          const int s = sk & 1;
#ifdef DI_PROF_CONV3
          long long t0 = clock64();
#endif
          mbar_wait(&sfull[s], (sk >> 1) & 1);
#ifdef DI_PROF_CONV3
          c_s += clock64() - t0;
#endif
          tc_fence_after();
          for (int t = 0; t < ntiles; ++t) {
            const int tt = ti + t, a = tt % NACC;
            if (h == 0 && tt >= NACC) {
#ifdef DI_PROF_CONV3
              long long t1 = clock64();
#endif
              mbar_wait(&acc_empty[a], ((tt / NACC) - 1) & 1);
#ifdef DI_PROF_CONV3
              c_a += clock64() - t1;
#endif
              tc_fence_after();
            }
            const uint32_t d = tmem + a * 64;
            uint64_t bd = bdesc_base + (uint64_t)((s * strip_alloc + t * OUT3 * 64) >> 4);
            const uint64_t a0 = adesc0 + (uint64_t)((h * W3_BYTES) >> 4);
#pragma unroll
            for (int tu = 0; tu < 11; ++tu) {
              const uint64_t ad = a0 + (uint64_t)((tu * 2048) >> 4);
              if (TF32) {
                umma_ws_tf32(d, ad, bd, idesc, (h | tu) != 0);
                umma_ws_tf32(d, ad + 2, bd + 2, idesc, 1);   // second K=8 chunk: +32 B
              } else {
                umma_ws_f16(d, ad, bd, idesc, tu != 0);
                umma_ws_f16(d, ad + 2, bd + 2, idesc, 1);    // second K=16 half: +32 B
              }
              bd += bstep;
            }
            if (h == NH - 1) umma_commit(&acc_full[a]);
          }
          umma_commit(&sempty[s]);
        }
        ti += ntiles;
#ifdef DI_PROF_CONV3
        ++it;
#endif
      }
#ifdef DI_PROF_CONV3
      if (blockIdx.x % 37 == 0)
        printf("conv3 cta %d issuer: cycles %lld strip-wait %lld acc-wait %lld units %d tiles %d\n", blockIdx.x,
               clock64() - c0_, c_s, c_a, it, ti);
#endif
    }
  } else if (warp >= 4) {  // ---------------------------------------------- epilogue
    const int q = warp - 4;
    const int e = threadIdx.x - 128;
    int ti = 0;
    const float bsc = (!fullmap && bias) ? bias[0] : 0.f;
    for (int u = blockIdx.x; u < g.units; u += gridDim.x) {
      const int b = u / per_img, rem = u - b * per_img;
      const int r0 = (rem / g.ncs) * g.R, c0 = (rem % g.ncs) * g.wseg;
      const int rows = min(g.R, g.n1 - r0);
      const int L = (rows - 1) * P + g.wseg;
      for (int n0 = 0; n0 < L; n0 += OUT3, ++ti) {
        const int cnt = min(OUT3, L - n0);
        const int a = ti % NACC;
        mbar_wait(&acc_full[a], (ti / NACC) & 1);
        tc_fence_after();
        const uint32_t taddr = tmem + a * 64 + ((uint32_t)(q * 32) << 16);
        uint32_t r0v[32], r1v[32];
        tmem_ld32(taddr, r0v);
        tmem_ld32(taddr + 32, r1v);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[a]);
        if (lane < 11) {
          float* dst = S + lane * SROW + 64 * q;
#pragma unroll
          for (int j = 0; j < 32; ++j) dst[j] = __uint_as_float(r0v[j]);
#pragma unroll
          for (int j = 0; j < 32; ++j) dst[32 + j] = __uint_as_float(r1v[j]);
        }
        named_bar(1, 128);
        for (int orel = e; orel < cnt; orel += 128) {
          float acc = 0.f;
#pragma unroll
          for (int v = 0; v < 11; ++v) acc += S[v * SROW + orel + v];
          const int o = n0 + orel;
          const int rr = o / P, cc = o - rr * P;
          if (cc < g.wseg && c0 + cc < g.n2 && rr < rows) {
            const size_t pix = ((size_t)b * g.n1 + r0 + rr) * g.n2 + c0 + cc;
            acc += (fullmap && bias) ? bias[pix % ((size_t)g.n1 * g.n2)] : bsc;
            if (relu) acc = fmaxf(acc, 0.f);
            xhat[pix] = acc;
          }
        }
        named_bar(1, 128);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<256>(tmem);
}

// =============================================================================================== host
static Geo13 make_geo13(int batch, int n1, int n2, int R, bool conv1) {
  Geo13 g;
  g.n1 = n1, g.n2 = n2, g.R = R;
  g.wseg = n2 < 64 ? n2 : 64;
  g.P = conv1 ? ((g.wseg + 10 + 7) & ~7) : g.wseg + 10;
  g.nrb = ceil_div(n1, R);
  g.ncs = ceil_div(n2, g.wseg);
  g.units = batch * g.nrb * g.ncs;
  g.guard = 0;
  return g;
}

size_t conv1_tc_smem_bytes() { return (size_t)C1_STAGE_OFF + 8 * 2 * C1_STAGE + 1024; }

// finite guard rows past a conv3 strip: the last tile's last K-block reads positions up to
// (ntiles - 1) * OUT3 + 10 P + 255 of a (R + 10) P-position strip
static int conv3_guard(int wseg) {
  const int P = wseg + 10, L = (R3 - 1) * P + wseg, nt = ceil_div(L, OUT3);
  const int need = (nt - 1) * OUT3 + 10 * P + 256 - (R3 + 10) * P;
  return (need > 0 ? need : 0) + 8;
}

size_t conv3_tc_smem_bytes(int n2, bool tf32) {
  const int wseg = n2 < 64 ? n2 : 64, P = wseg + 10;
  const size_t strip_alloc = ((size_t)(R3 + 10) * P * 64 + (size_t)conv3_guard(wseg) * 64 + 1023) & ~(size_t)1023;
  return (size_t)(tf32 ? 2 : 1) * W3_BYTES + 2 * strip_alloc + 11 * SROW * 4 + 1024;
}
int conv3_tc_box_rows() { return R3 + 10; }
int conv3_tc_box_ch(bool tf32) { return tf32 ? 16 : 32; }
int conv3_tc_box_cols(int n2) { return (n2 < 64 ? n2 : 64) + 10; }

size_t conv1_tf32_smem_bytes() { return (size_t)W1T_BYTES + 2 * IM_BYTES_T + 2 * XT_STRIDE + 1024; }
int conv1_tf32_box_rows() { return R1T + 10; }

cudaError_t launch_conv1_tf32(const CUtensorMap* tmX, const void* w1pack, const float* bias, int fullmap, float* h1,
                              int batch, int n1, int n2, int num_sms, cudaStream_t st) {
  Geo13 g = make_geo13(batch, n1, n2, R1T, true);
  const int grid = g.units < num_sms ? g.units : num_sms;
  k_conv1_tf32<64, false><<<grid, 384, conv1_tf32_smem_bytes(), st>>>(*tmX, reinterpret_cast<const uint8_t*>(w1pack),
                                                                      bias, fullmap, g, h1, nullptr, 0, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_conv1g_tf32(int cout, const CUtensorMap* tmX, const void* w1pack, const float* bias, float* out,
                               int batch, int n1, int n2, int num_sms, cudaStream_t st) {
  if (cout == 64) return launch_conv1_tf32(tmX, w1pack, bias, 0, out, batch, n1, n2, num_sms, st);
  if (cout != 32) return cudaErrorInvalidValue;
  Geo13 g = make_geo13(batch, n1, n2, R1T, true);
  const int grid = g.units < num_sms ? g.units : num_sms;
  k_conv1_tf32<32, false><<<grid, 384, conv1_tf32_smem_bytes(), st>>>(*tmX, reinterpret_cast<const uint8_t*>(w1pack),
                                                                      bias, 0, g, out, nullptr, 0, nullptr);
  return cudaGetLastError();
}

// dG2 = [h2 > 0] * dgrad3(dG3) written in bf16 (dg2b: the operand of wgrad2 and dgrad2) and the layer-2 bias
// gradient gb2[32] = sum of dG2 (per-CTA partials in part_b, then a fixed-order fp64 reduction)
cudaError_t launch_dgrad3_tf32(const CUtensorMap* tmDX, const void* wpack, const void* h2, void* dg2b, float* part_b,
                               float* gb2, int batch, int n1, int n2, int num_sms, cudaStream_t st, bool h2_bf16) {
  Geo13 g = make_geo13(batch, n1, n2, R1T, true);
  const int grid = g.units < num_sms ? g.units : num_sms;
  k_conv1_tf32<32, true><<<grid, 384, conv1_tf32_smem_bytes(), st>>>(*tmDX, reinterpret_cast<const uint8_t*>(wpack),
                                                                     nullptr, 0, g, reinterpret_cast<float*>(dg2b), h2,
                                                                     h2_bf16 ? 1 : 0, part_b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_bias_reduce(part_b, grid, 32, gb2, st);
}

cudaError_t setup_conv13_tc(int n2) {
  cudaError_t e0 = cudaFuncSetAttribute(k_conv1_tf32<64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)conv1_tf32_smem_bytes());
  if (e0 != cudaSuccess) return e0;
  e0 = cudaFuncSetAttribute(k_conv1_tf32<32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)conv1_tf32_smem_bytes());
  if (e0 != cudaSuccess) return e0;
  e0 = cudaFuncSetAttribute(k_conv1_tf32<32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)conv1_tf32_smem_bytes());
  if (e0 != cudaSuccess) return e0;
  cudaError_t e = cudaFuncSetAttribute(k_conv1_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)conv1_tc_smem_bytes());
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_conv1_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)conv1_tc_smem_bytes());
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_conv3_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)conv3_tc_smem_bytes(n2, false));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_conv3_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)conv3_tc_smem_bytes(n2, true));
}

int conv1_tc_box_rows() { return R1 + 10; }
int conv1_tc_box_cols(int n2) { return (((n2 < 64 ? n2 : 64) + 10 + 7) & ~7) + 8; }

// tmS (may be null): the TMA store map over h1 (encode_h1_store: box 16 ch x 64 cols x 2 rows, SWIZZLE_32B)
cudaError_t launch_conv1_tc(const CUtensorMap* tmX, const CUtensorMap* tmS, const void* xt, const void* w1pack,
                            const float* bias, int fullmap, void* h1, int batch, int n1, int n2, int num_sms,
                            cudaStream_t st) {
  Geo13 g = make_geo13(batch, n1, n2, R1, true);
  const int grid = g.units < num_sms ? g.units : num_sms;
  auto k = tmX ? k_conv1_tc<true> : k_conv1_tc<false>;
  CUtensorMap dummy{};
  return launch_ex(k, dim3(grid), dim3(384), conv1_tc_smem_bytes(), st, 1, true, tmX ? *tmX : dummy,
                   tmS ? *tmS : dummy, tmS ? 1 : 0, reinterpret_cast<const __nv_bfloat16*>(xt),
                   reinterpret_cast<const uint8_t*>(w1pack), bias, fullmap, g, reinterpret_cast<__nv_bfloat16*>(h1));
}

cudaError_t launch_conv3_tc(const CUtensorMap* tmH2, const void* w3pack, const float* bias, int fullmap, int relu,
                            float* xhat, int batch, int n1, int n2, int num_sms, bool tf32, cudaStream_t st) {
  Geo13 g = make_geo13(batch, n1, n2, R3, false);
  g.guard = conv3_guard(g.wseg);
  const int grid = g.units < num_sms ? g.units : num_sms;
  auto k = tf32 ? k_conv3_tc<true> : k_conv3_tc<false>;
  k<<<grid, 256, conv3_tc_smem_bytes(n2, tf32), st>>>(*tmH2, reinterpret_cast<const uint8_t*>(w3pack), bias,
                                                      fullmap, relu, g, xhat);
  return cudaGetLastError();
}

DI_DEBUG_BINDER(di_debug_bind_k_conv13_tc)

}  // namespace di
