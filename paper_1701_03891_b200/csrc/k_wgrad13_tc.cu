// k_wgrad13_tc.cu -- training: the weight gradients of the THIN layers on tcgen05.
//
//   layer 1 (C_in = 1):  dwx1[co][a][b] = sum_p dG1[p][co] * x~[p + (a-5, b-5)]           (k_train.cu header)
//                        (dG1 arrives in bf16 from the bf16 layer-2 dgrad; its bias sum is taken over those values)
//   layer 3 (C_out = 1): dwx3[ci][a][b] = sum_p dG3[p]     * h2[p + (a-5, b-5)][ci]
//
// Both contract over pixel positions with one single-channel operand.  As in k_wgrad2_tc.cu the operands are
// MN-major bf16 tiles (kind::f16; tf32 cannot read MN-major), fp32 accumulation in TMEM over all the CTA's work
// units, and the taps are descriptor strides -- plus, for the single-channel map, a shared-memory TOEPLITZ
// EXPANSION: row q of E holds the 16 values map[q + j] (j = 0..15, a 32-B row, SWIZZLE_32B), so that E viewed
// as an MN-major operand with atoms P rows apart is the (row tap, column tap) x position matrix of the map:
//   layer 1: A = E(x~) (M = 8 row taps x 16 column taps, atom i = row tap a0 + i at LBO = P rows of E),
//            B = dG1 strip (SWIZZLE_128B, N = 64 channels), two MMAs per 16 positions (a0 = 0 and a0 = 3; the
//            rows a = 3..7 of the second are duplicates and discarded);
//   layer 3: A = h2 strip (SWIZZLE_64B, M = 4 row taps x 32 channels, atoms P positions apart),
//            B = E'(dG3) with E'[k][j] = dG3[k - j] (N = 16 column taps), three MMAs per 16 positions
//            (a0 = 0, 4, 7; a = 7 of the third is discarded).
// The gradient operand (dG1 / dG3) covers only the unit's own output pixels (origin (r0, c0), zero in the 10
// trailing columns of each P-position row), the activation operand (x~ / h2) carries the 5-pixel halo (origin
// (r0 - 5, c0 - 5)), so position p + a P + b is pixel p shifted by (a - 5, b - 5) without wrapping into the next
// row, and every (pixel, tap) product is counted once.  Work units are
// double-buffered: the 128 threads convert unit i+1 (fp32 -> bf16, swizzled) while the MMAs of unit i run.
// Bias gradients (sum of the fp32 dG over pixels) are summed by the loading threads in a fixed assignment.
// Per-CTA partials are reduced in fp64 in a fixed order (deterministic).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.cuh"
#define DI_TU_ID 8
#include "sm100.cuh"

namespace di {

namespace {
constexpr int R = WG13_ROWS;      // output rows per unit
constexpr int WSEG = 64;
constexpr int KS = 11;

struct GeoT13 {
  int n1, n2, wseg, P, nrb, ncs, units;
  int off2, stage;                // second region offset, stage bytes
};

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&t);
}

// layer 1 stage: [dG1: 16 lead + R*P + 32 guard positions x 128 B] [E: 32 lead + NE + 32 guard rows x 32 B]
__host__ __device__ inline int l1_ne(int P) { return (R + 11) * P + 16; }
__host__ __device__ inline int l1_nx(int P) { return l1_ne(P) + 16; }
// layer 3 stage: [h2: 16 lead + NH + 32 guard positions x 64 B] [E': 32 lead + NB + 32 guard rows x 32 B]
__host__ __device__ inline int l3_nh(int P) { return (R + 11) * P + 32; }
__host__ __device__ inline int l3_nb(int P) { return R * P + 32; }
}  // namespace

// =============================================================================================== layer 1
__global__ void __launch_bounds__(128, 1)
    k_wgrad1_tc(const void* __restrict__ xt, const __nv_bfloat16* __restrict__ dg1, GeoT13 g,
                float* __restrict__ part, float* __restrict__ part_b, int xbf, const __grid_constant__ CUtensorMap tmD1,
                int use_tma) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  float* xs = reinterpret_cast<float*>(smem + 2 * g.stage);
  __shared__ uint64_t done[2], fin, dbar[2];
  __shared__ uint32_t tslot;
  __shared__ float red[128][9];
  const int tid = threadIdx.x, warp = warp_id(), lane = lane_id();
  const int P = g.P, NE = l1_ne(P), NX = l1_nx(P);
  if (tid == 0) {
    mbar_init(&done[0], 1), mbar_init(&done[1], 1), mbar_init(&fin, 1);
    mbar_init(&dbar[0], 1), mbar_init(&dbar[1], 1);
    if (use_tma) tma_prefetch_desc(&tmD1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<128>(&tslot), tmem_relinquish();
  for (int s = 0; s < 2; ++s) {   // zero every stage once: leads / guards are never rewritten
    uint4* p = reinterpret_cast<uint4*>(smem + s * g.stage);
    for (int i = tid; i < g.stage / 16; i += 128) p[i] = make_uint4(0, 0, 0, 0);
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int per_img = g.nrb * g.ncs;
  const int cg = tid & 7;   // fixed 8-channel group of this thread's dG1 chunks (bias partials)
  float bs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const uint32_t id = idesc_f32acc(1, 128, 64, 1, 1);
  // this thread's x~ halo-strip values of unit un: q = tid + 128 uu (NX <= 17 * 74 + 32 <= 128 XPT)
  constexpr int XPT = 11;
  uint32_t xv[XPT];   // raw bits (bf16 zero-extended, or fp32): converted only where they are stored, so the loads
                      // stay in flight until then
  auto load_x = [&](int un, uint32_t* v) {
    const int bb = un / per_img, rm = un - bb * per_img;
    const int rr0 = (rm / g.ncs) * R, cc0 = (rm % g.ncs) * g.wseg;
#pragma unroll
    for (int uu = 0; uu < XPT; ++uu) {
      const int q = tid + uu * 128, row = q / P, col = q - row * P;
      const int gr = rr0 - 5 + row, gc = cc0 - 5 + col;
      const size_t xi = ((size_t)bb * g.n1 + gr) * g.n2 + gc;
      v[uu] = (q < NX && gr >= 0 && gr < g.n1 && gc >= 0 && gc < g.n2)
                  ? (xbf ? (uint32_t)__ldg(reinterpret_cast<const unsigned short*>(xt) + xi)
                         : __ldg(reinterpret_cast<const uint32_t*>(xt) + xi))
                  : 0u;
    }
  };
  int it = 0;
  uint32_t acc = 0;
  for (int u = blockIdx.x; u < g.units; u += gridDim.x, ++it) {
    const int s = it & 1;
    const int b = u / per_img, rem = u - b * per_img;
    const int r0 = (rem / g.ncs) * R, c0 = (rem % g.ncs) * g.wseg;
    const int rows = min(R, g.n1 - r0);
    uint8_t* d1 = smem + s * g.stage;          // position q at d1 + (16 + q) * 128
    uint8_t* ex = smem + s * g.stage + g.off2;  // row q at ex + (32 + q) * 32
    if (it >= 2) mbar_wait(&done[s], ((it >> 1) - 1) & 1);
    // dG1 of the unit's pixels: position q -> (r0 + q / P, c0 + q % P), columns >= wseg zero; bf16 SW128.
    // use_tma: one TMA box of R rows x P columns (out-of-bounds zero fill); the columns of the next segment are
    // zeroed and the bias sums read back from shared memory once it has landed (below)
    if (use_tma && tid == 0) {
      mbar_arrive_expect_tx(&dbar[s], (uint32_t)(R * P * 128));
      tma_load_4d(d1 + 16 * 128, &tmD1, &dbar[s], 0, c0, r0, b);
    }
    constexpr int U = 4;   // chunks per thread in flight (memory-level parallelism)
    for (int i0 = tid; !use_tma && i0 < R * P * 8; i0 += 128 * U) {
      uint4 v[U];
#pragma unroll
      for (int uu = 0; uu < U; ++uu) {
        const int i = i0 + uu * 128, q = i >> 3, row = q / P, col = q - row * P;
        const int gr = r0 + row, gc = c0 + col;
        v[uu] = make_uint4(0, 0, 0, 0);
        if (i < R * P * 8 && row < rows && col < g.wseg && gc < g.n2)
          v[uu] = __ldg(reinterpret_cast<const uint4*>(dg1 + (((size_t)b * g.n1 + gr) * g.n2 + gc) * 64 + 8 * cg));
      }
#pragma unroll
      for (int uu = 0; uu < U; ++uu) {
        const int i = i0 + uu * 128, q = i >> 3;
        if (i >= R * P * 8) break;
        const uint4 w = v[uu];
        bs[0] += __uint_as_float(w.x << 16), bs[1] += __uint_as_float(w.x & 0xffff0000u);
        bs[2] += __uint_as_float(w.y << 16), bs[3] += __uint_as_float(w.y & 0xffff0000u);
        bs[4] += __uint_as_float(w.z << 16), bs[5] += __uint_as_float(w.z & 0xffff0000u);
        bs[6] += __uint_as_float(w.w << 16), bs[7] += __uint_as_float(w.w & 0xffff0000u);
        *reinterpret_cast<uint4*>(d1 + (16 + q) * 128 + ((cg ^ (q & 7)) << 4)) = w;
      }
    }
    // x~ strip with halo: xs[q] = x~(r0 - 5 + q / P, c0 - 5 + q % P), loaded into registers one unit ahead
    if (it == 0) load_x(u, xv);
#pragma unroll
    for (int uu = 0; uu < XPT; ++uu)
      if (tid + uu * 128 < NX) xs[tid + uu * 128] = __uint_as_float(xbf ? xv[uu] << 16 : xv[uu]);
    if (use_tma) {
      mbar_wait(&dbar[s], (it >> 1) & 1);
      if (g.ncs > 1)   // columns wseg .. P-1 of each row belong to the next segment
        for (int i = tid; i < R * (P - g.wseg) * 8; i += 128) {
          const int row = i / ((P - g.wseg) * 8), rr = i % ((P - g.wseg) * 8);
          const int q = row * P + g.wseg + rr / 8;
          *reinterpret_cast<uint4*>(d1 + (16 + q) * 128 + ((rr % 8) << 4)) = make_uint4(0, 0, 0, 0);
        }
      __syncthreads();
      for (int q = tid >> 3; q < rows * P; q += 16) {   // bias partials: channel group cg, fixed assignment
        const uint4 w = *reinterpret_cast<const uint4*>(d1 + (16 + q) * 128 + ((cg ^ (q & 7)) << 4));
        bs[0] += __uint_as_float(w.x << 16), bs[1] += __uint_as_float(w.x & 0xffff0000u);
        bs[2] += __uint_as_float(w.y << 16), bs[3] += __uint_as_float(w.y & 0xffff0000u);
        bs[4] += __uint_as_float(w.z << 16), bs[5] += __uint_as_float(w.z & 0xffff0000u);
        bs[6] += __uint_as_float(w.w << 16), bs[7] += __uint_as_float(w.w & 0xffff0000u);
      }
    }
    __syncthreads();
    // Toeplitz expansion E[q][j] = xs[q + j], SW32 (16-B chunk c at c ^ ((q >> 2) & 1))
    for (int i = tid; i < 2 * NE; i += 128) {
      const int q = i >> 1, c = i & 1;
      const float* x = xs + q + 8 * c;
      *reinterpret_cast<uint4*>(ex + (32 + q) * 32 + ((c ^ ((q >> 2) & 1)) << 4)) =
          make_uint4(pack2(x[0], x[1]), pack2(x[2], x[3]), pack2(x[4], x[5]), pack2(x[6], x[7]));
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const int nk = (rows * P + 15) >> 4;
      uint64_t bd = smem_desc(smem_u32(d1 + 16 * 128), 128, 1024, kSwizzle128B);
      uint64_t a1 = smem_desc(smem_u32(ex + 32 * 32), P * 32, 256, kSwizzle32B);
      uint64_t a2 = smem_desc(smem_u32(ex + (32 + 3 * P) * 32), P * 32, 256, kSwizzle32B);
      for (int k = 0; k < nk; ++k, bd += 128, a1 += 32, a2 += 32) {   // +16 positions
        umma_f16_ss(tmem, a1, bd, id, acc);
        umma_f16_ss(tmem + 64, a2, bd, id, acc);
        acc = 1;
      }
      umma_commit(&done[s]);
    }
    if (u + (int)gridDim.x < g.units) load_x(u + gridDim.x, xv);   // in flight across the MMAs and the next TMA wait
    __syncthreads();   // xs is rewritten by the next unit's loaders
  }
  if (tid == 0) umma_commit(&fin);
  mbar_wait(&fin, 0);
  tc_fence_after();
  float* dst = part + ((size_t)blockIdx.x * 128 + warp * 32 + lane) * 128;
  for (int c = 0; c < 128; c += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 16; j += 4)
      *reinterpret_cast<float4*>(dst + c + j) = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                                            __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) red[tid][j] = bs[j];
  __syncthreads();
  if (tid < 64) {   // channel 8 cg' + j: threads with tid % 8 == cg', in order
    const int c8 = tid >> 3, j = tid & 7;
    float t = 0.f;
    for (int r = c8; r < 128; r += 8) t += red[r][j];
    part_b[(size_t)blockIdx.x * 64 + tid] = t;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<128>(tmem);
}

// gw1 [64][11][11] (API orientation), gb1 [64]
// Deterministic sums over the CTA partials: a block owns 32 consecutive partial elements (coalesced reads) x 8 slices
// of the CTA index, combined in a fixed order in fp64.  L = 1: part [c][128][128] (m = tap slot, n = co / 64 + co),
// L = 3: part [c][128][48]; blockIdx.y = 1 sums the bias partials (part_b [c][nb]).
template <int L>
__global__ void __launch_bounds__(256) k_wgrad13_reduce(const float* __restrict__ part, const float* __restrict__ part_b,
                                                        int nct, int flip, float* __restrict__ gw,
                                                        float* __restrict__ gb) {
  constexpr int NCOLS = L == 1 ? 128 : 48, E = 128 * NCOLS, NB = L == 1 ? 64 : 1;
  __shared__ double sh[8][33];
  const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;
  const bool bias = blockIdx.y == 1;
  const int e = blockIdx.x * 32 + lx, ne = bias ? NB : E;
  if (bias && blockIdx.x * 32 >= NB) return;
  const float* p = (bias ? part_b : part) + e;
  double t = 0.0;
  if (e < ne)
    for (int c = ly; c < nct; c += 8) t += p[(size_t)c * ne];
  sh[ly][lx] = t;
  __syncthreads();
  if (ly != 0 || e >= ne) return;
  for (int k = 1; k < 8; ++k) t += sh[k][lx];
  if (bias) {
    gb[e] = (float)t;
    return;
  }
  const int m = e / NCOLS, n = e % NCOLS;
  int a, bb, ch;
  if (L == 1) {   // m = a * 16 + bb (a <= 7, n = co) or (a - 3) * 16 + bb (a >= 8, n = 64 + co)
    bb = m % 16, ch = n % 64;
    a = n < 64 ? m / 16 : m / 16 + 3;
    if (bb >= KS || (n >= 64 && a < 8) || a >= KS) return;
  } else {        // m = ii * 32 + ci, n = grp * 16 + bb; a = ii (grp 0), 4 + ii (grp 1), 7 + ii (grp 2, ii >= 1)
    const int grp = n / 16, ii = m / 32;
    bb = n % 16, ch = m % 32;
    a = grp == 0 ? ii : grp == 1 ? 4 + ii : 7 + ii;
    if (bb >= KS || (grp == 2 && ii == 0)) return;
  }
  gw[(size_t)ch * KS * KS + (flip ? (KS - 1 - a) * KS + (KS - 1 - bb) : a * KS + bb)] = (float)t;
}

// =============================================================================================== layer 3
__global__ void __launch_bounds__(128, 1)
    k_wgrad3_tc(const void* __restrict__ h2, const float* __restrict__ dg3, GeoT13 g, float* __restrict__ part,
                float* __restrict__ part_b, int hbf, const __grid_constant__ CUtensorMap tmH2, int use_tma) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  float* ds = reinterpret_cast<float*>(smem + 2 * g.stage) + 16;   // ds[-16 .. NB + 16)
  __shared__ uint64_t done[2], fin, hbar[2];
  __shared__ uint32_t tslot;
  __shared__ float red[128];
  const int tid = threadIdx.x, warp = warp_id(), lane = lane_id();
  const int P = g.P, NH = l3_nh(P), NB = l3_nb(P);
  if (tid == 0) {
    mbar_init(&done[0], 1), mbar_init(&done[1], 1), mbar_init(&fin, 1);
    mbar_init(&hbar[0], 1), mbar_init(&hbar[1], 1);
    if (use_tma) tma_prefetch_desc(&tmH2);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<64>(&tslot), tmem_relinquish();
  for (int s = 0; s < 2; ++s) {
    uint4* p = reinterpret_cast<uint4*>(smem + s * g.stage);
    for (int i = tid; i < g.stage / 16; i += 128) p[i] = make_uint4(0, 0, 0, 0);
  }
  for (int i = tid; i < NB + 32; i += 128) ds[i - 16] = 0.f;
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int per_img = g.nrb * g.ncs;
  float bsum = 0.f;
  const uint32_t id = idesc_f32acc(1, 128, 16, 1, 1);
  int it = 0;
  uint32_t acc = 0;
  for (int u = blockIdx.x; u < g.units; u += gridDim.x, ++it) {
    const int s = it & 1;
    const int b = u / per_img, rem = u - b * per_img;
    const int r0 = (rem / g.ncs) * R, c0 = (rem % g.ncs) * g.wseg;
    const int rows = min(R, g.n1 - r0);
    uint8_t* hs = smem + s * g.stage;          // position q at hs + (16 + q) * 64
    uint8_t* ex = smem + s * g.stage + g.off2;  // row k at ex + (32 + k) * 32
    if (it >= 2) mbar_wait(&done[s], ((it >> 1) - 1) & 1);
    // h2 strip with halo: q -> h2(r0 - 5 + q / P, c0 - 5 + q % P), bf16 SW64 (chunk c at c ^ ((q >> 1) & 3));
    // bf16 h2 (BF16 contexts): one TMA box of R + 11 rows (out-of-bounds zero fill), else converting loaders
    if (use_tma && tid == 0) {
      mbar_arrive_expect_tx(&hbar[s], (uint32_t)((R + 11) * P * 64));
      tma_load_4d(hs + 16 * 64, &tmH2, &hbar[s], 0, c0 - 5, r0 - 5, b);
    }
    constexpr int U = 4;
    for (int i0 = tid; !use_tma && i0 < NH * 4; i0 += 128 * U) {
      uint4 w[U];   // 8 channels of one position as bf16
#pragma unroll
      for (int uu = 0; uu < U; ++uu) {
        const int i = i0 + uu * 128, q = i >> 2, c = i & 3, row = q / P, col = q - row * P;
        const int gr = r0 - 5 + row, gc = c0 - 5 + col;
        w[uu] = make_uint4(0, 0, 0, 0);
        if (i < NH * 4 && gr >= 0 && gr < g.n1 && gc >= 0 && gc < g.n2) {
          const size_t off = (((size_t)b * g.n1 + gr) * g.n2 + gc) * 32 + 8 * c;
          if (hbf) {
            w[uu] = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(h2) + off));
          } else {
            const float4* src = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(h2) + off);
            const float4 v0 = __ldg(src), v1 = __ldg(src + 1);
            w[uu] = make_uint4(pack2(v0.x, v0.y), pack2(v0.z, v0.w), pack2(v1.x, v1.y), pack2(v1.z, v1.w));
          }
        }
      }
#pragma unroll
      for (int uu = 0; uu < U; ++uu) {
        const int i = i0 + uu * 128, q = i >> 2, c = i & 3;
        if (i >= NH * 4) break;
        *reinterpret_cast<uint4*>(hs + (16 + q) * 64 + ((c ^ ((q >> 1) & 3)) << 4)) = w[uu];
      }
    }
    // dG3 of the unit's own pixels (zero elsewhere): ds[p], p -> (r0 + p / P, c0 + p % P)
    for (int p0 = tid; p0 < R * P; p0 += 128 * 4) {
      float v[4];
#pragma unroll
      for (int uu = 0; uu < 4; ++uu) {
        const int p = p0 + uu * 128, row = p / P, col = p - row * P;
        const int gc = c0 + col;
        v[uu] = (p < R * P && row < rows && col < g.wseg && gc < g.n2)
                    ? __ldg(dg3 + ((size_t)b * g.n1 + r0 + row) * g.n2 + gc) : 0.f;
      }
#pragma unroll
      for (int uu = 0; uu < 4; ++uu)
        if (p0 + uu * 128 < R * P) bsum += v[uu], ds[p0 + uu * 128] = v[uu];
    }
    __syncthreads();
    // E'[k][j] = ds[k - j], SW32
    for (int i = tid; i < 2 * NB; i += 128) {
      const int k = i >> 1, c = i & 1;
      const float* x = ds + k - 8 * c;   // j = 8c .. 8c + 7 -> ds[k - j]
      *reinterpret_cast<uint4*>(ex + (32 + k) * 32 + ((c ^ ((k >> 2) & 1)) << 4)) =
          make_uint4(pack2(x[0], x[-1]), pack2(x[-2], x[-3]), pack2(x[-4], x[-5]), pack2(x[-6], x[-7]));
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      if (use_tma) mbar_wait(&hbar[s], (it >> 1) & 1);
      tc_fence_after();
      const int nk = (rows * P + 11 + 15) >> 4;
      uint64_t bd = smem_desc(smem_u32(ex + 32 * 32), 32, 256, kSwizzle32B);
      uint64_t a0 = smem_desc(smem_u32(hs + 16 * 64), P * 64, 512, kSwizzle64B);
      uint64_t a1 = smem_desc(smem_u32(hs + (16 + 4 * P) * 64), P * 64, 512, kSwizzle64B);
      uint64_t a2 = smem_desc(smem_u32(hs + (16 + 7 * P) * 64), P * 64, 512, kSwizzle64B);
      for (int k = 0; k < nk; ++k, bd += 32, a0 += 64, a1 += 64, a2 += 64) {   // +16 positions
        umma_f16_ss(tmem, a0, bd, id, acc);
        umma_f16_ss(tmem + 16, a1, bd, id, acc);
        umma_f16_ss(tmem + 32, a2, bd, id, acc);
        acc = 1;
      }
      umma_commit(&done[s]);
    }
    __syncthreads();   // ds is rewritten by the next unit
  }
  if (tid == 0) umma_commit(&fin);
  mbar_wait(&fin, 0);
  tc_fence_after();
  float* dst = part + ((size_t)blockIdx.x * 128 + warp * 32 + lane) * 48;
  for (int c = 0; c < 48; c += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 16; j += 4)
      *reinterpret_cast<float4*>(dst + c + j) = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                                            __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
  }
  red[tid] = bsum;
  __syncthreads();
  if (tid == 0) {
    float t = 0.f;
    for (int r = 0; r < 128; ++r) t += red[r];
    part_b[blockIdx.x] = t;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<64>(tmem);
}

// gw3 [32][11][11] (API orientation of W3 [1][32][11][11]), gb3 [1]
// =============================================================================================== host
static GeoT13 make_geo(int batch, int n1, int n2, bool l1) {
  GeoT13 g;
  g.n1 = n1, g.n2 = n2;
  g.wseg = n2 < WSEG ? n2 : WSEG;
  g.P = g.wseg + 10;
  g.nrb = (n1 + R - 1) / R;
  g.ncs = (n2 + g.wseg - 1) / g.wseg;
  g.units = batch * g.nrb * g.ncs;
  int r1, r2;
  if (l1) {
    r1 = (16 + R * g.P + 32) * 128;
    r2 = (32 + l1_ne(g.P) + 32) * 32;
  } else {
    r1 = (16 + l3_nh(g.P) + 32) * 64;
    r2 = (32 + l3_nb(g.P) + 32) * 32;
  }
  g.off2 = (r1 + 1023) & ~1023;
  g.stage = (g.off2 + r2 + 1023) & ~1023;
  return g;
}

static size_t smem_bytes(int n2, bool l1) {
  GeoT13 g = make_geo(1, 1, n2, l1);
  const size_t extra = l1 ? (size_t)(l1_nx(g.P) + 16) * 4 : (size_t)(l3_nb(g.P) + 48) * 4;
  return 2 * (size_t)g.stage + extra + 1024;
}

size_t wgrad13_tc_part_floats(int num_sms) { return (size_t)num_sms * 128 * 128; }

cudaError_t setup_wgrad13_tc(int n2) {
  cudaError_t e = cudaFuncSetAttribute(k_wgrad1_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem_bytes(n2, true));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_wgrad3_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes(n2, false));
}

int wgrad1_tc_d_box_rows() { return R; }

cudaError_t launch_wgrad1_tc(const void* xt, const void* dg1, int batch, int n1, int n2, float* part, float* part_b,
                             int flip, float* gw, float* gb, int num_sms, cudaStream_t st, bool xt_bf16,
                             const CUtensorMap* tmD1) {
  GeoT13 g = make_geo(batch, n1, n2, true);
  const int grid = g.units < num_sms ? g.units : num_sms;
  CUtensorMap dummy{};
  k_wgrad1_tc<<<grid, 128, smem_bytes(n2, true), st>>>(xt, reinterpret_cast<const __nv_bfloat16*>(dg1), g, part,
                                                       part_b, xt_bf16 ? 1 : 0, tmD1 ? *tmD1 : dummy,
                                                       tmD1 ? 1 : 0);
  k_wgrad13_reduce<1><<<dim3(128 * 128 / 32, 2), 256, 0, st>>>(part, part_b, grid, flip, gw, gb);
  return cudaGetLastError();
}

int wgrad3_tc_h_box_rows() { return R + 11; }

cudaError_t launch_wgrad3_tc(const void* h2, const float* dg3, int batch, int n1, int n2, float* part, float* part_b,
                             int flip, float* gw, float* gb, int num_sms, cudaStream_t st, bool h2_bf16,
                             const CUtensorMap* tmH2) {
  GeoT13 g = make_geo(batch, n1, n2, false);
  const int grid = g.units < num_sms ? g.units : num_sms;
  CUtensorMap dummy{};
  const int use_tma = (h2_bf16 && tmH2) ? 1 : 0;
  k_wgrad3_tc<<<grid, 128, smem_bytes(n2, false), st>>>(h2, dg3, g, part, part_b, h2_bf16 ? 1 : 0,
                                                        use_tma ? *tmH2 : dummy, use_tma);
  k_wgrad13_reduce<3><<<dim3(128 * 48 / 32, 2), 256, 0, st>>>(part, part_b, grid, flip, gw, gb);
  return cudaGetLastError();
}

DI_DEBUG_BINDER(di_debug_bind_k_wgrad13_tc)

}  // namespace di
