// k_wgrad2_tc.cu -- training: the layer-2 weight gradient on tcgen05, and the bf16
// operand staging it reads.
//
//   dwx2[co][ci][a][b] = sum_{images, p} dG2[p][co] * H1[p + (a-5, b-5)][ci]          (k_train.cu header)
//
// is a contraction over PIXELS: K = pixel positions, one GEMM per tap.  Both operands are stored pixel-major
// (NHWC), i.e. MN-major for this contraction; tcgen05 reads MN-major operands for kind::f16 (bf16) but not for
// kind::tf32 (tools/scratch/mnmajor.cu: tf32 MN-major yields zeros), so the operands are bf16 copies of h1 and dG2
// with fp32 accumulation.  The taps become strides of the shared-memory descriptors, no im2col:
//   * A = the h1 strip (SWIZZLE_128B, one 128-B row = 64 channels per position), M = 128 = two row taps
//     (a0, a0 + 1) x 64 ci: the second M atom sits P positions (one strip row) after the first (LBO = P * 128 B);
//   * B = the dG2 strip (SWIZZLE_64B, one 64-B row = 32 channels per position), N = 32 x (column taps): N atom t
//     is the same strip shifted by ONE position (LBO = 64 B, overlapping atoms), so one MMA covers 8 column taps;
//   * K steps of 16 positions walk the flattened (row, column) positions of the unit's dG2 rows; the dG2 strip's
//     halo columns are zero (TMA out-of-bounds fill, or zeroed in smem when the image is split in column
//     segments), so a flattened shift equals the 2-D shift.
// TMEM holds the accumulators of one ROLE = row-tap pair (a0 = 2 role): columns [0, 256) for b = 7..0 (8 atoms),
// [256, 352) for b = 10..8 (3 atoms).  Six roles cover a = 0..11 (a = 11 is discarded).  CTAs are assigned
// (role, unit subset) and accumulate over all their units; the epilogue dumps the 128 x 352 partial, and
// k_wgrad2_reduce sums the partials of a role in a fixed order in fp64 (deterministic).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.cuh"
#define DI_TU_ID 9
#include "sm100.cuh"

namespace di {

namespace {
constexpr int R = WG2_ROWS;        // dG2 rows per unit
constexpr int WSEG = 64;
constexpr int NROLE = 6;
constexpr int NCOL = 352;          // TMEM accumulator columns per role
constexpr int KS = 11;

struct GeoW {
  int n1, n2, wseg, P, nrb, ncs, units, nper;
  int offG, stage;                 // dG2 region offset inside a stage, stage bytes
};

__host__ __device__ inline int h_bytes(int P) { return (R + 1) * P * 128; }
__host__ __device__ inline int g_bytes(int P) { return R * P * 64; }
}  // namespace

// stage layout: [1024 zero][h1 box (R+1) x P x 128 B][32 x 128 B zero] | [1024 zero][dG2 box R x P x 64 B][32 x 64 zero]
__global__ void __launch_bounds__(128, 1)
    k_wgrad2_tc(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmG, GeoW g,
                float* __restrict__ part) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  __shared__ uint64_t full[2], ready[2], empty[2], done;
  __shared__ uint32_t tslot;
  const int warp = warp_id(), lane = lane_id();
  const int role = blockIdx.x % NROLE, idx = blockIdx.x / NROLE;
  const int a0 = 2 * role;
  const int hb = h_bytes(g.P), gb = g_bytes(g.P);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmH), tma_prefetch_desc(&tmG);
    for (int s = 0; s < 2; ++s) mbar_init(&full[s], 1), mbar_init(&ready[s], 1), mbar_init(&empty[s], 1);
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&tslot), tmem_relinquish();
  for (int s = 0; s < 2; ++s) {   // zero leads and guards once (TMA never writes them)
    uint8_t* st = smem + s * g.stage;
    for (int i = threadIdx.x; i < 64; i += blockDim.x) reinterpret_cast<uint4*>(st)[i] = make_uint4(0, 0, 0, 0);
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
      reinterpret_cast<uint4*>(st + 1024 + hb)[i] = make_uint4(0, 0, 0, 0);
    for (int i = threadIdx.x; i < 64; i += blockDim.x)
      reinterpret_cast<uint4*>(st + g.offG)[i] = make_uint4(0, 0, 0, 0);
    for (int i = threadIdx.x; i < 128; i += blockDim.x)
      reinterpret_cast<uint4*>(st + g.offG + 1024 + gb)[i] = make_uint4(0, 0, 0, 0);
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int per_img = g.nrb * g.ncs;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ producer
      int it = 0;
      for (int u = idx; u < g.units; u += g.nper, ++it) {
        const int s = it & 1;
        const int b = u / per_img, rem = u - b * per_img;
        const int r0 = (rem / g.ncs) * R, c0 = (rem % g.ncs) * g.wseg;
        if (it >= 2) mbar_wait(&empty[s], ((it >> 1) - 1) & 1);
        uint8_t* st = smem + s * g.stage;
        mbar_arrive_expect_tx(&full[s], hb + gb);
        tma_load_4d(st + 1024, &tmH, &full[s], 0, c0 - 5, r0 - 5 + a0, b);
        tma_load_4d(st + g.offG + 1024, &tmG, &full[s], 0, c0 - 5, r0, b);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      const uint32_t id1 = idesc_f32acc(1, 128, 256, 1, 1), id2 = idesc_f32acc(1, 128, 96, 1, 1);
      int it = 0;
      uint32_t acc = 0;
      for (int u = idx; u < g.units; u += g.nper, ++it) {
        const int s = it & 1;
        const int rem = u % per_img;
        const int rows = min(R, g.n1 - (rem / g.ncs) * R);
        const int nk = (rows * g.P + 8 + 15) >> 4;
        mbar_wait(g.ncs > 1 ? &ready[s] : &full[s], (it >> 1) & 1);
        tc_fence_after();
        const uint32_t hbase = smem_u32(smem + s * g.stage + 1024), gbase = smem_u32(smem + s * g.stage + g.offG + 1024);
        // A: h1 box position (-6 | -3) + k; B: dG2 box position -8 + t + k (see header)
        uint64_t a1 = smem_desc(hbase - 6 * 128, g.P * 128, 1024, kSwizzle128B);
        uint64_t a2 = smem_desc(hbase - 3 * 128, g.P * 128, 1024, kSwizzle128B);
        uint64_t bd = smem_desc(gbase - 8 * 64, 64, 512, kSwizzle64B);
        for (int k = 0; k < nk; ++k, a1 += 128, a2 += 128, bd += 64) {   // +16 positions per step
          umma_f16_ss(tmem, a1, bd, id1, acc);
          umma_f16_ss(tmem + 256, a2, bd, id2, acc);
          acc = 1;
        }
        umma_commit(&empty[s]);
      }
      umma_commit(&done);
    }
  } else if (warp == 2) {  // ------------------------------------------- halo-column fixup (column segments)
    if (g.ncs > 1) {
      int it = 0;
      for (int u = idx; u < g.units; u += g.nper, ++it) {
        const int s = it & 1;
        mbar_wait(&full[s], (it >> 1) & 1);
        uint8_t* gs = smem + s * g.stage + g.offG + 1024;
        for (int i = lane; i < R * 10 * 4; i += 32) {   // R rows x 10 halo positions x 4 chunks of 16 B
          const int row = i / 40, j = (i % 40) / 4, ch = i % 4;
          const int col = j < 5 ? j : g.wseg + j;
          reinterpret_cast<uint4*>(gs + (row * g.P + col) * 64)[ch] = make_uint4(0, 0, 0, 0);
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ready[s]);
      }
    }
  }
  // ------------------------------------------------------------------ epilogue: all four warps, lanes 32w..
  __syncwarp();
  mbar_wait(&done, 0);
  tc_fence_after();
  float* dst = part + ((size_t)(role * g.nper + idx) * 128 + warp * 32 + lane) * NCOL;
  for (int c = 0; c < NCOL; c += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 16; j += 4)
      *reinterpret_cast<float4*>(dst + c + j) =
          make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                      __uint_as_float(r[j + 3]));
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// gw (API orientation, [co][ci][u][v]) = sum over the role's CTAs (fp64, fixed order).  A block owns 32 consecutive
// partial elements (coalesced reads) x 8 slices of the CTA index; the slices are combined in a fixed order.
__global__ void __launch_bounds__(256) k_wgrad2_reduce(const float* __restrict__ part, int nper, int flip,
                                                       float* __restrict__ gw) {
  constexpr int E = 128 * NCOL;
  __shared__ double sh[8][33];
  const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5, role = blockIdx.y;
  const int e = blockIdx.x * 32 + lx;
  const float* p = part + (size_t)role * nper * E + e;
  double t = 0.0;
  if (e < E)
    for (int c = ly; c < nper; c += 8) t += p[(size_t)c * E];
  sh[ly][lx] = t;
  __syncthreads();
  if (ly != 0 || e >= E) return;
  for (int k = 1; k < 8; ++k) t += sh[k][lx];
  const int m = e / NCOL, n = e % NCOL;
  const int a = role * 2 + m / 64, ci = m % 64;
  if (a >= KS) return;                                  // row tap 11 of the last role: discarded
  const int b = n < 256 ? 7 - n / 32 : 10 - (n - 256) / 32, co = n % 32;
  gw[((size_t)co * 64 + ci) * KS * KS + (flip ? (KS - 1 - a) * KS + (KS - 1 - b) : a * KS + b)] = (float)t;
}

// fp32 -> bf16 copy (n multiple of 8)
__global__ void k_to_bf16(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, size_t n8) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n8; i += (size_t)gridDim.x * blockDim.x) {
    const float4 a = reinterpret_cast<const float4*>(src)[2 * i], b = reinterpret_cast<const float4*>(src)[2 * i + 1];
    uint4 o;
    __nv_bfloat162 t;
    t = __floats2bfloat162_rn(a.x, a.y), o.x = *reinterpret_cast<uint32_t*>(&t);
    t = __floats2bfloat162_rn(a.z, a.w), o.y = *reinterpret_cast<uint32_t*>(&t);
    t = __floats2bfloat162_rn(b.x, b.y), o.z = *reinterpret_cast<uint32_t*>(&t);
    t = __floats2bfloat162_rn(b.z, b.w), o.w = *reinterpret_cast<uint32_t*>(&t);
    reinterpret_cast<uint4*>(dst)[i] = o;
  }
}

// dG2 fp32 [pix][32] -> bf16, and the per-block channel sums of the fp32 values (bias gradient partials,
// part_b[block][32]); grid = WGRAD_CHUNKS blocks of 256 threads, thread = (pixel slot, 8-channel group)
__global__ void __launch_bounds__(256) k_dg2_bf16(const float* __restrict__ dg, size_t npix,
                                                  __nv_bfloat16* __restrict__ dst, float* __restrict__ part_b) {
  const int q = threadIdx.x & 3;
  float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const size_t n8 = npix * 4;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n8; i += (size_t)gridDim.x * blockDim.x) {
    const float4 a = reinterpret_cast<const float4*>(dg)[2 * i], b = reinterpret_cast<const float4*>(dg)[2 * i + 1];
    s[0] += a.x, s[1] += a.y, s[2] += a.z, s[3] += a.w, s[4] += b.x, s[5] += b.y, s[6] += b.z, s[7] += b.w;
    uint4 o;
    __nv_bfloat162 t;
    t = __floats2bfloat162_rn(a.x, a.y), o.x = *reinterpret_cast<uint32_t*>(&t);
    t = __floats2bfloat162_rn(a.z, a.w), o.y = *reinterpret_cast<uint32_t*>(&t);
    t = __floats2bfloat162_rn(b.x, b.y), o.z = *reinterpret_cast<uint32_t*>(&t);
    t = __floats2bfloat162_rn(b.z, b.w), o.w = *reinterpret_cast<uint32_t*>(&t);
    reinterpret_cast<uint4*>(dst)[i] = o;
  }
  __shared__ float red[256][9];
#pragma unroll
  for (int j = 0; j < 8; ++j) red[threadIdx.x][j] = s[j];
  __syncthreads();
  if (threadIdx.x < 32) {   // channel c = 8 q' + j: sum over the 64 threads with that q', in thread order
    const int qq = threadIdx.x / 8, j = threadIdx.x % 8;
    float t = 0.f;
    for (int r = qq; r < 256; r += 4) t += red[r][j];
    part_b[(size_t)blockIdx.x * 32 + threadIdx.x] = t;
  }
  (void)q;
}

static GeoW make_geo_w(int batch, int n1, int n2, int num_sms) {
  GeoW g;
  g.n1 = n1, g.n2 = n2;
  g.wseg = n2 < WSEG ? n2 : WSEG;
  g.P = g.wseg + 10;
  g.nrb = (n1 + R - 1) / R;
  g.ncs = (n2 + g.wseg - 1) / g.wseg;
  g.units = batch * g.nrb * g.ncs;
  g.nper = num_sms / NROLE;
  if (g.nper > g.units) g.nper = g.units;
  if (g.nper < 1) g.nper = 1;
  const int hreg = (1024 + h_bytes(g.P) + 32 * 128 + 1023) & ~1023;
  const int greg = (1024 + g_bytes(g.P) + 32 * 64 + 1023) & ~1023;
  g.offG = hreg;
  g.stage = hreg + greg;
  return g;
}

size_t wgrad2_tc_smem_bytes(int n2) { return 2 * (size_t)make_geo_w(1, 1, n2, NROLE).stage + 1024; }
int wgrad2_tc_h_box_rows() { return R + 1; }
int wgrad2_tc_g_box_rows() { return R; }
size_t wgrad2_tc_part_floats(int num_sms) { return (size_t)NROLE * (num_sms / NROLE) * 128 * NCOL; }

cudaError_t setup_wgrad2_tc(int n2) {
  return cudaFuncSetAttribute(k_wgrad2_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wgrad2_tc_smem_bytes(n2));
}

cudaError_t launch_wgrad2_tc(const CUtensorMap* tmH, const CUtensorMap* tmG, int batch, int n1, int n2, float* part,
                             int flip, float* gw, int num_sms, cudaStream_t st) {
  GeoW g = make_geo_w(batch, n1, n2, num_sms);
  k_wgrad2_tc<<<NROLE * g.nper, 128, wgrad2_tc_smem_bytes(n2), st>>>(*tmH, *tmG, g, part);
  k_wgrad2_reduce<<<dim3(128 * NCOL / 32, NROLE), 256, 0, st>>>(part, g.nper, flip, gw);
  return cudaGetLastError();
}

cudaError_t launch_to_bf16(const float* src, void* dst, size_t n, cudaStream_t st) {
  k_to_bf16<<<4 * 148, 256, 0, st>>>(src, reinterpret_cast<__nv_bfloat16*>(dst), n / 8);
  return cudaGetLastError();
}

cudaError_t launch_dg2_bf16(const float* dg, size_t npix, void* dst, float* part_b, cudaStream_t st) {
  k_dg2_bf16<<<WGRAD_CHUNKS, 256, 0, st>>>(dg, npix, reinterpret_cast<__nv_bfloat16*>(dst), part_b);
  return cudaGetLastError();
}

DI_DEBUG_BINDER(di_debug_bind_k_wgrad2_tc)

}  // namespace di
