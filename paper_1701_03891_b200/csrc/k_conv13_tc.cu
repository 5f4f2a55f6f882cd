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
// Roles (256 threads): warp 0 producer (weights once; conv3: TMA strips), warp 1 single-thread MMA issuer,
// warps 2-3 conv1 im2row builders (warp 2 also allocates TMEM), warps 4-7 epilogue (TMEM lane quadrants).
// Strips / im2row buffers are double-buffered across units; accumulators rotate over 4 TMEM slots.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "sm100.cuh"

namespace di {

namespace {
constexpr int NACC = 4;

struct Geo13 {
  int n1, n2, wseg, P, R, nrb, ncs, units;
};

__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------- conv1 geometry
constexpr int R1 = C1TC_ROWS;           // output rows per unit
constexpr int P1MAX = 80;
constexpr int IM_ROWS = R1 * P1MAX + 256 + 10 * P1MAX;   // im2row rows per buffer (>= ntiles*256 + 10P)
constexpr int IM_BYTES = IM_ROWS * 32;
constexpr int STRIP_WORDS = (IM_ROWS + 32) / 2;          // strip_lin as words (zero past the real strip)
constexpr int SW1_OFF = ((STRIP_WORDS + 31) & ~31) + 16;  // word offset of the one-element-shifted copy
constexpr int FILL_PER_THREAD = ((R1 + 10) * P1MAX + 63) / 64;   // strip elements per builder thread
constexpr int W1_BYTES = 11 * 64 * 32;                   // 11 tap rows x 64 filters x 16 taps bf16

// ---------------------------------------------------------------- conv3 geometry
constexpr int R3 = C3TC_ROWS;
constexpr int OUT3 = 256 - 10;
constexpr int GUARD3 = 256;                              // finite rows past the strip (see below)
constexpr int W3_BYTES = 11 * 32 * 64;                   // 11 tap rows x 32 (v) rows x 32 ch bf16
constexpr int SROW = 267;                                // S row stride (floats), odd -> conflict-free
}  // namespace

// =============================================================================================== conv1
__global__ void __launch_bounds__(256, 1)
    k_conv1_tc(const __nv_bfloat16* __restrict__ xt, const uint8_t* __restrict__ w1pack,
               const float* __restrict__ bias, int fullmap, Geo13 g, __nv_bfloat16* __restrict__ h1) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* wbuf = smem;                                           // 22 KB
  uint8_t* const im0 = smem + W1_BYTES;   // 2 x 54 KB im2row buffers (1024-aligned: W1_BYTES = 22528)
  uint32_t* const sw0 = reinterpret_cast<uint32_t*>(smem + W1_BYTES + 2 * IM_BYTES);
  uint32_t* const sw1 = sw0 + SW1_OFF;

  __shared__ uint64_t wbar, im_full[2], im_empty[2], acc_full[NACC], acc_empty[NACC];
  __shared__ uint32_t tslot;
  const int warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    mbar_init(&wbar, 1);
    for (int s = 0; s < 2; ++s) mbar_init(&im_full[s], 64), mbar_init(&im_empty[s], 1);
    for (int a = 0; a < NACC; ++a) mbar_init(&acc_full[a], 1), mbar_init(&acc_empty[a], 4);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&tslot), tmem_relinquish();
  for (int i = threadIdx.x; i < 2 * SW1_OFF; i += blockDim.x) sw0[i] = 0u;   // zero tails of both copies
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int per_img = g.nrb * g.ncs;
  const int P = g.P;

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
      int it = 0, ti = 0;
      for (int u = blockIdx.x; u < g.units; u += gridDim.x, ++it) {
        const int rem = u % per_img;
        const int r0 = (rem / g.ncs) * g.R;
        const int rows = min(g.R, g.n1 - r0);
        const int L = (rows - 1) * P + g.wseg;
        const int s = it & 1;
        mbar_wait(&im_full[s], (it >> 1) & 1);
        tc_fence_after();
        for (int n0 = 0; n0 < L; n0 += 256, ++ti) {
          const int cnt = min(256, L - n0);
          const int N = cnt > 128 ? 256 : (cnt > 64 ? 128 : 64);
          const uint32_t idesc = idesc_f32acc(1, 64, N);
          const int a = ti % NACC;
          if (ti >= NACC) mbar_wait(&acc_empty[a], ((ti / NACC) - 1) & 1);
          tc_fence_after();
          const uint32_t d = tmem + a * 128;
          uint64_t bd = bdesc_base + (uint64_t)(((s * IM_BYTES) + n0 * 32) >> 4);
          const uint64_t bstep = (uint64_t)((P * 32) >> 4);
#pragma unroll
          for (int tu = 0; tu < 11; ++tu) {
            umma_ws_f16(d, adesc0 + (uint64_t)((tu * 2048) >> 4), bd, idesc, tu != 0);
            bd += bstep;
          }
          umma_commit(&acc_full[a]);
        }
        umma_commit(&im_empty[s]);
      }
    }
  } else if (warp < 4) {  // ------------------------------------------- im2row builders (64 threads)
    // strip_lin[idx] = x_tilde[b][r0-5+rr][c0-5+cc] (zero outside the image and past the 5-px halo), kept twice
    // as 32-bit words: sw0 = strip_lin, sw1 = strip_lin shifted by one element, so that the 16-element window
    // of ANY row m is 8 aligned words (from sw0 if m is even, sw1 if odd).  sw1 sits 16 words (mod 32) after
    // sw0: a warp's 32 consecutive rows read 32 distinct banks.
    const int bt = threadIdx.x - 64;
    uint16_t* s0 = reinterpret_cast<uint16_t*>(sw0);
    uint16_t* s1 = reinterpret_cast<uint16_t*>(sw1);
    int it = 0;
    for (int u = blockIdx.x; u < g.units; u += gridDim.x, ++it) {
      const int b = u / per_img, rem = u - b * per_img;
      const int r0 = (rem / g.ncs) * g.R, c0 = (rem % g.ncs) * g.wseg;
      const int s = it & 1;
      if (it >= 2) mbar_wait(&im_empty[s], ((it >> 1) - 1) & 1);
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
      // im2row: row m = strip_lin[m .. m+15], SWIZZLE_32B (16-B chunk h of row m at m*32 + ((h ^ (m>>2 & 1)) << 4))
      uint8_t* dst = im0 + s * IM_BYTES;
      for (int m = bt; m < IM_ROWS; m += 64) {
        const uint32_t* w = ((m & 1) ? sw1 : sw0) + (m >> 1);
        const int sw = (m >> 2) & 1;
        *reinterpret_cast<uint4*>(dst + m * 32 + (sw << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
        *reinterpret_cast<uint4*>(dst + m * 32 + ((1 ^ sw) << 4)) = make_uint4(w[4], w[5], w[6], w[7]);
      }
      fence_async_smem();
      mbar_arrive(&im_full[s]);
      named_bar(2, 64);  // the strip is refilled for the next unit only after every builder is done reading it
    }
  } else {  // -------------------------------------------------------- epilogue, warps 4..7
    const int q = warp - 4;
    const int f = 32 * (q & 1) + lane;  // filter (TMEM lane within the quadrant)
    __nv_bfloat16* tw = reinterpret_cast<__nv_bfloat16*>(sw0 + 2 * SW1_OFF) + q * 32 * 32;   // 2 KB per warp
    const float bch = (!fullmap && bias) ? bias[f] : 0.f;
    int ti = 0;
    for (int u = blockIdx.x; u < g.units; u += gridDim.x) {
      const int b = u / per_img, rem = u - b * per_img;
      const int r0 = (rem / g.ncs) * g.R, c0 = (rem % g.ncs) * g.wseg;
      const int rows = min(g.R, g.n1 - r0);
      const int L = (rows - 1) * P + g.wseg;
      for (int n0 = 0; n0 < L; n0 += 256, ++ti) {
        const int cnt = min(256, L - n0);
        const int N = cnt > 128 ? 256 : (cnt > 64 ? 128 : 64);
        const int half = N / 2;
        const int a = ti % NACC;
        mbar_wait(&acc_full[a], (ti / NACC) & 1);
        tc_fence_after();
        const uint32_t taddr = tmem + a * 128 + ((uint32_t)(q * 32) << 16);
        const int pbase = n0 + (q >> 1) * half;
        for (int c = 0; c < half; c += 32) {
          uint32_t r[32];
          tmem_ld32(taddr + c, r);
          tmem_ld_wait();
          // position o0 + j of the strip -> (row rr, column cc); j < 32 < P wraps at most once
          const int o0 = pbase + c;
          const int rr0 = o0 / P, cc0 = o0 - rr0 * P;
          // (1) bias + ReLU + bf16, transposed through this warp's smem tile T[j][channel] (64-B rows)
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float bv = bch;
            if (fullmap && bias) {
              int cc = cc0 + j, rr = rr0;
              if (cc >= P) cc -= P, ++rr;
              const int gy = min(r0 + rr, g.n1 - 1), gx = min(c0 + cc, g.n2 - 1);
              bv = bias[((size_t)gy * g.n2 + gx) * 64 + f];
            }
            tw[j * 32 + lane] = __float2bfloat16_rn(fmaxf(__uint_as_float(r[j]) + bv, 0.f));
          }
          __syncwarp();
          // (2) 16-B coalesced NHWC stores: thread -> (position j = lane/4 + 8i, 8-channel chunk k = lane%4)
          const uint4* t4 = reinterpret_cast<const uint4*>(tw);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int j = (lane >> 2) + 8 * i, k = lane & 3;
            int cc = cc0 + j, rr = rr0;
            if (cc >= P) cc -= P, ++rr;
            if (o0 + j < n0 + cnt && cc < g.wseg && c0 + cc < g.n2 && rr < rows) {
              const size_t pix = ((size_t)b * g.n1 + r0 + rr) * g.n2 + c0 + cc;
              *reinterpret_cast<uint4*>(h1 + pix * 64 + 32 * (q & 1) + 8 * k) = t4[j * 4 + k];
            }
          }
          __syncwarp();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[a]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// =============================================================================================== conv3
__global__ void __launch_bounds__(256, 1)
    k_conv3_tc(const __grid_constant__ CUtensorMap tmH2, const uint8_t* __restrict__ w3pack,
               const float* __restrict__ bias, int fullmap, int relu, Geo13 g, float* __restrict__ xhat) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int P = g.P;
  const int strip_bytes = (g.R + 10) * P * 64;
  const int strip_alloc = (strip_bytes + GUARD3 * 64 + 1023) & ~1023;
  uint8_t* wbuf = smem;                                       // 22 KB (1024-aligned size: 22528)
  uint8_t* const strip0 = smem + W3_BYTES;  // 2 strip buffers, strip_alloc apart
  float* S = reinterpret_cast<float*>(smem + W3_BYTES + 2 * strip_alloc);   // [11][SROW]

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
  // Guard rows after each strip: the B windows of the last tile of a unit read up to 245 rows past the
  // TMA box (their outputs are discarded), but 0 * NaN would not be: keep them finite.
  for (int s = 0; s < 2; ++s)
    for (int i = threadIdx.x; i < GUARD3 * 64 / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(strip0 + s * strip_alloc + strip_bytes)[i] = make_uint4(0, 0, 0, 0);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int per_img = g.nrb * g.ncs;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ producer
      mbar_arrive_expect_tx(&wbar, W3_BYTES);
      bulk_load(wbuf, w3pack, W3_BYTES, &wbar);
      int it = 0;
      for (int u = blockIdx.x; u < g.units; u += gridDim.x, ++it) {
        const int b = u / per_img, rem = u - b * per_img;
        const int r0 = (rem / g.ncs) * g.R, c0 = (rem % g.ncs) * g.wseg;
        const int s = it & 1;
        if (it >= 2) mbar_wait(&sempty[s], ((it >> 1) - 1) & 1);
        mbar_arrive_expect_tx(&sfull[s], strip_bytes);
        tma_load_4d(strip0 + s * strip_alloc, &tmH2, &sfull[s], 0, c0 - 5, r0 - 5, b);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      mbar_wait(&wbar, 0);
      tc_fence_after();
      constexpr uint32_t idesc = idesc_f32acc(1, 32, 256);
      const uint64_t adesc0 = smem_desc(smem_u32(wbuf), 16, 512, kSwizzle64B);
      const uint64_t bdesc_base = smem_desc(smem_u32(strip0), 16, 512, kSwizzle64B);
      const uint64_t bstep = (uint64_t)((P * 64) >> 4);
      int it = 0, ti = 0;
      for (int u = blockIdx.x; u < g.units; u += gridDim.x, ++it) {
        const int rem = u % per_img;
        const int r0 = (rem / g.ncs) * g.R;
        const int rows = min(g.R, g.n1 - r0);
        const int L = (rows - 1) * P + g.wseg;
        const int s = it & 1;
        mbar_wait(&sfull[s], (it >> 1) & 1);
        tc_fence_after();
        for (int n0 = 0; n0 < L; n0 += OUT3, ++ti) {
          const int a = ti % NACC;
          if (ti >= NACC) mbar_wait(&acc_empty[a], ((ti / NACC) - 1) & 1);
          tc_fence_after();
          const uint32_t d = tmem + a * 64;
          uint64_t bd = bdesc_base + (uint64_t)((s * strip_alloc + n0 * 64) >> 4);
#pragma unroll
          for (int tu = 0; tu < 11; ++tu) {
            const uint64_t ad = adesc0 + (uint64_t)((tu * 2048) >> 4);
            umma_ws_f16(d, ad, bd, idesc, tu != 0);
            umma_ws_f16(d, ad + 2, bd + 2, idesc, 1);   // second K=16 half: +32 B
            bd += bstep;
          }
          umma_commit(&acc_full[a]);
        }
        umma_commit(&sempty[s]);
      }
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
  return g;
}

size_t conv1_tc_smem_bytes() { return (size_t)W1_BYTES + 2 * IM_BYTES + 2 * SW1_OFF * 4 + 4 * 2048 + 1024; }

size_t conv3_tc_smem_bytes(int n2) {
  const int wseg = n2 < 64 ? n2 : 64, P = wseg + 10;
  const size_t strip_alloc = ((size_t)(R3 + 10) * P * 64 + GUARD3 * 64 + 1023) & ~(size_t)1023;
  return (size_t)W3_BYTES + 2 * strip_alloc + 11 * SROW * 4 + 1024;
}
int conv3_tc_box_rows() { return R3 + 10; }
int conv3_tc_box_cols(int n2) { return (n2 < 64 ? n2 : 64) + 10; }

cudaError_t setup_conv13_tc(int n2) {
  cudaError_t e = cudaFuncSetAttribute(k_conv1_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)conv1_tc_smem_bytes());
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_conv3_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)conv3_tc_smem_bytes(n2));
}

cudaError_t launch_conv1_tc(const void* xt, const void* w1pack, const float* bias, int fullmap, void* h1, int batch,
                            int n1, int n2, int num_sms, cudaStream_t st) {
  Geo13 g = make_geo13(batch, n1, n2, R1, true);
  const int grid = g.units < num_sms ? g.units : num_sms;
  k_conv1_tc<<<grid, 256, conv1_tc_smem_bytes(), st>>>(reinterpret_cast<const __nv_bfloat16*>(xt),
                                                       reinterpret_cast<const uint8_t*>(w1pack), bias, fullmap, g,
                                                       reinterpret_cast<__nv_bfloat16*>(h1));
  return cudaGetLastError();
}

cudaError_t launch_conv3_tc(const CUtensorMap* tmH2, const void* w3pack, const float* bias, int fullmap, int relu,
                            float* xhat, int batch, int n1, int n2, int num_sms, cudaStream_t st) {
  Geo13 g = make_geo13(batch, n1, n2, R3, false);
  const int grid = g.units < num_sms ? g.units : num_sms;
  k_conv3_tc<<<grid, 256, conv3_tc_smem_bytes(n2), st>>>(*tmH2, reinterpret_cast<const uint8_t*>(w3pack), bias,
                                                         fullmap, relu, g, xhat);
  return cudaGetLastError();
}

}  // namespace di
