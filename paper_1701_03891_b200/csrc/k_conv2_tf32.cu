// k_conv2_tf32.cu -- the 11x11 multi-channel convolutions in TF32 mode (fp32 activations, tcgen05.mma kind::tf32,
// fp32 accumulation), one template for every (C_in, C_out) in {32, 64} x {32, 64}:
//   * stage 2 of the paper's stack, conv layer 2 (64 -> 32, bias + ReLU, crop S);
//   * (EPI_MASK: a ReLU'-masked data gradient; the training step runs its layer-2 one on the bf16 kernel instead);
//   * the interior layers of deeper / wider stacks.
//
// Same implicit-GEMM mapping as the bf16 kernel (k_conv2_tc.cu): pixels are the UMMA N dimension, TAPS = 128 / C_out
// column taps v' x C_out filters stack into M = 128, the B operand is a window of a zero-padded shared-memory strip
// and output o receives sum_v' D[v'*C_out + k][o - n0 + v'].  What differs from bf16:
//   * an fp32 position row of 32 channels is one 128-B swizzle row, so the K dimension is split into C_in / 32
//     channel halves h; K-block = (h, u, v0 = TAPS j): 11 * ceil(11 / TAPS) per half, 4 MMAs of K = 8 each;
//   * the strip holds ONE channel half ((R + 10) rows x P positions x 128 B, one 4-D TMA box at channel 32h) and
//     is reloaded per half;
//   * both tiles of a unit (<= 2 for R = 6) accumulate at once (TMEM columns [0, 256) and [256, 512)) so each
//     16-KB weight block serves both tiles; the epilogue runs between units, two warp groups (one per tile).
// Weight block (h, u, j): row v'*C_out + k, 32 fp32 channels 32h + c, SWIZZLE_128B (api.cu conv_tf32_pack).
#include <cuda_runtime.h>

#include "kernels.cuh"
#define DI_TU_ID 5
#include "sm100.cuh"

namespace di {

namespace {
constexpr int R = C2_ROWS;             // output rows per unit (6)
constexpr int WSEG = 64;
constexpr int NT = 256;
constexpr int OUT_PER_TILE = NT - 3;   // 253 (>= TAPS - 1 columns of slack for every C_out)
constexpr int WSTAGES = 3;             // 3 x 16 KB: room for two epilogue groups' staging
constexpr uint32_t WBYTES = C2_KBLOCK_BYTES;  // 16 KB: 128 rows x 32 fp32 channels
constexpr int GUARD_ROWS = 24;
constexpr int SPS = 36;
constexpr int ECH = 16;

struct GeoT {
  int n1, n2, wseg, P, nrb, ncs, units;
};
}  // namespace

__device__ __forceinline__ void ld_tail13_t(uint32_t taddr, uint32_t* r) {
  tmem_ld8(taddr, r);
  tmem_ld4(taddr + 8, r + 8);
  tmem_ld1(taddr + 12, r + 12);
}

enum { EPI_BIAS_RELU = 0, EPI_MASK = 1 };

// MODE EPI_BIAS_RELU: out = ReLU(conv + bias) (per-channel bias, or full-map bias [n1*n2][C_out] when fullmap);
// MODE EPI_MASK:      out = [mask > 0] * conv (the ReLU' of the layer whose gradient this is)
template <int CIN, int COUT, int MODE>
__global__ void __launch_bounds__(384, 1)
    k_conv_tf32(const __grid_constant__ CUtensorMap tmIn, const float* __restrict__ wpack,
                const float* __restrict__ bias, int fullmap, const float* __restrict__ mask, GeoT g,
                float* __restrict__ out) {
  constexpr int TAPS = 128 / COUT;            // column taps stacked in M
  constexpr int J = (11 + TAPS - 1) / TAPS;   // column-tap groups per tap row
  constexpr int KBH = 11 * J;                 // K-blocks per channel half
  constexpr int BOXC = 32;                    // fp32 channels per strip row (one 128-B swizzle row)
  constexpr int RB = BOXC * 4;                // strip / weight row bytes
  constexpr int NH = CIN / BOXC;              // channel halves
  constexpr int KMMA = RB / 32;               // MMAs per K-block (32 B of K each)
  constexpr uint32_t WB = 128 * RB;           // weight block bytes
  constexpr uint32_t SWZ = RB == 128 ? kSwizzle128B : kSwizzle64B;
  constexpr int QPT = COUT / 32;              // TMEM lane quadrants per tap
  constexpr int CPT = COUT / 8;               // channels per epilogue thread
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align_smem_1024(smem_raw);
  const int strip_bytes = (R + 10) * g.P * RB;
  const int strip_alloc = (strip_bytes + GUARD_ROWS * RB + 1023) & ~1023;
  uint8_t* strip = smem;
  uint8_t* wst = smem + strip_alloc;
  float* sP = reinterpret_cast<float*>(wst + WSTAGES * WB);

  __shared__ uint64_t sfull, sempty, wfull[WSTAGES], wempty[WSTAGES], tfull, tempty;
  __shared__ uint32_t tslot;
  const int warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmIn);
    mbar_init(&sfull, 1), mbar_init(&sempty, 1);
    for (int s = 0; s < WSTAGES; ++s) mbar_init(&wfull[s], 1), mbar_init(&wempty[s], 1);
    mbar_init(&tfull, 1), mbar_init(&tempty, 8);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&tslot), tmem_relinquish();
  for (int i = threadIdx.x; i < GUARD_ROWS * RB / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(strip + strip_bytes)[i] = make_uint4(0, 0, 0, 0);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int per_img = g.nrb * g.ncs;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ producer: strips + weights, in order
      uint32_t wk = 0, sk = 0;
      for (int u = blockIdx.x; u < g.units; u += gridDim.x) {
        const int b = u / per_img, rem = u - b * per_img;
        const int r0 = (rem / g.ncs) * R, c0 = (rem % g.ncs) * g.wseg;
        for (int h = 0; h < NH; ++h, ++sk) {
          if (sk > 0) mbar_wait(&sempty, (sk - 1) & 1);
          mbar_arrive_expect_tx(&sfull, strip_bytes);
          tma_load_4d(strip, &tmIn, &sfull, BOXC * h, c0 - 5, r0 - 5, b);
          const uint8_t* wsrc = reinterpret_cast<const uint8_t*>(wpack) + (size_t)h * KBH * WB;
          for (int kb = 0; kb < KBH; ++kb, ++wk, wsrc += WB) {
            const uint32_t st = wk % WSTAGES;
            if (wk >= WSTAGES) mbar_wait(&wempty[st], ((wk / WSTAGES) - 1) & 1);
            mbar_arrive_expect_tx(&wfull[st], WB);
            bulk_load(wst + st * WB, wsrc, WB, &wfull[st]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      const uint64_t bdesc0 = smem_desc(smem_u32(strip), 16, 8 * RB, SWZ);
      const uint64_t adesc0 = smem_desc(smem_u32(wst), 16, 8 * RB, SWZ);
      const uint64_t pstep = (uint64_t)g.P * (RB >> 4);
      uint32_t wk = 0, sk = 0;
      int it = 0;
      for (int u = blockIdx.x; u < g.units; u += gridDim.x, ++it) {
        const int rem = u % per_img;
        const int r0 = (rem / g.ncs) * R;
        const int rows = min(R, g.n1 - r0);
        const int L = (rows - 1) * g.P + g.wseg;
        const int ntiles = (L + OUT_PER_TILE - 1) / OUT_PER_TILE;   // 1 or 2
        const int nB = ntiles > 1 ? min(NT, (min(OUT_PER_TILE, L - OUT_PER_TILE) + TAPS - 1 + 15) & ~15) : 0;
        const int nA = min(NT, (min(OUT_PER_TILE, L) + TAPS - 1 + 15) & ~15);
        const uint32_t idA = idesc_f32acc(2, 128, nA), idB = idesc_f32acc(2, 128, nB > 0 ? nB : 16);
        if (it > 0) mbar_wait(&tempty, (it - 1) & 1);   // the epilogue drained the previous unit
        tc_fence_after();
        for (int h = 0; h < NH; ++h, ++sk) {
          mbar_wait(&sfull, sk & 1);
          tc_fence_after();
          uint64_t bd = bdesc0;
          for (int uu = 0; uu < 11; ++uu, bd += pstep) {
#pragma unroll
            for (int j = 0; j < J; ++j, ++wk) {
              const uint32_t st = wk % WSTAGES;
              mbar_wait(&wfull[st], (wk / WSTAGES) & 1);
              tc_fence_after();
              const uint64_t ad = adesc0 + (uint64_t)(st * (WB >> 4));
              const uint64_t b = bd + (uint64_t)(TAPS * j * (RB >> 4));   // v0 = TAPS j positions
              const uint32_t acc0 = (h | uu | j) != 0;
#pragma unroll
              for (int kk = 0; kk < KMMA; ++kk) umma_tf32_ss(tmem, ad + 2 * kk, b + 2 * kk, idA, kk ? 1u : acc0);
              if (nB > 0) {
                const uint64_t bb = b + (uint64_t)(OUT_PER_TILE * (RB >> 4));
#pragma unroll
                for (int kk = 0; kk < KMMA; ++kk) umma_tf32_ss(tmem + 256, ad + 2 * kk, bb + 2 * kk, idB, kk ? 1u : acc0);
              }
              umma_commit(&wempty[st]);
            }
          }
          umma_commit(&sempty);
        }
        umma_commit(&tfull);
      }
    }
  } else if (warp >= 4) {  // ---------------------------------------------- epilogue: group grp = tile grp
    const int q = warp & 3, grp = (warp - 4) >> 2;   // TMEM lane quadrant q = warp % 4: tap q / QPT
    const int shift = q / QPT;
    const int e = (threadIdx.x - 128) & 127;
    const int jj = e >> 3, kg = e & 7;               // output position jj of the chunk, channels CPT kg ..
    const int c0ch = CPT * kg, cblk = c0ch / 32, cl = c0ch % 32;
    float* const sPg = sP + grp * (4 * ECH * SPS);
    float bch[CPT];
#pragma unroll
    for (int i = 0; i < CPT; ++i) bch[i] = (MODE == EPI_BIAS_RELU && !fullmap && bias) ? bias[c0ch + i] : 0.f;
    int it = 0;
    for (int u = blockIdx.x; u < g.units; u += gridDim.x, ++it) {
      const int b = u / per_img, rem = u - b * per_img;
      const int r0 = (rem / g.ncs) * R, c0 = (rem % g.ncs) * g.wseg;
      const int rows = min(R, g.n1 - r0);
      const int L = (rows - 1) * g.P + g.wseg;
      const int ntiles = (L + OUT_PER_TILE - 1) / OUT_PER_TILE;
      mbar_wait(&tfull, it & 1);
      tc_fence_after();
      for (int t = grp; t < ntiles; t += 2) {
        const int n0 = t * OUT_PER_TILE;
        const int cnt = min(OUT_PER_TILE, L - n0);
        const uint32_t tq = tmem + t * 256 + ((uint32_t)(q * 32) << 16);
        for (int c = 0; c < cnt; c += ECH) {
          const int nout = min(ECH, cnt - c);
          uint32_t r[ECH];
          if (c + shift + ECH <= NT)
            tmem_ld16(tq + c + shift, r);
          else
            ld_tail13_t(tq + c + shift, r);
          tmem_ld_wait();
          float* dst = sPg + q * (ECH * SPS) + lane;
#pragma unroll
          for (int j = 0; j < ECH; ++j) dst[j * SPS] = __uint_as_float(r[j]);
          named_bar(1 + grp, 128);
          if (jj < nout) {
            const int o = n0 + c + jj;
            const int rr = o / g.P, cc = o - rr * g.P;
            if (cc < g.wseg && c0 + cc < g.n2 && rr < rows) {
              const size_t pix = ((size_t)b * g.n1 + r0 + rr) * g.n2 + c0 + cc;
#pragma unroll
              for (int v4 = 0; v4 < CPT / 4; ++v4) {
                float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int tp = 0; tp < TAPS; ++tp) {
                  const float4 a =
                      *reinterpret_cast<const float4*>(sPg + (tp * QPT + cblk) * (ECH * SPS) + jj * SPS + cl + 4 * v4);
                  sum.x += a.x, sum.y += a.y, sum.z += a.z, sum.w += a.w;
                }
                float* op = out + pix * COUT + c0ch + 4 * v4;
                if (MODE == EPI_MASK) {
                  const float4 m = __ldg(reinterpret_cast<const float4*>(mask + pix * COUT + c0ch + 4 * v4));
                  sum.x = m.x > 0.f ? sum.x : 0.f, sum.y = m.y > 0.f ? sum.y : 0.f;
                  sum.z = m.z > 0.f ? sum.z : 0.f, sum.w = m.w > 0.f ? sum.w : 0.f;
                } else {
                  float4 bv = make_float4(bch[4 * v4], bch[4 * v4 + 1], bch[4 * v4 + 2], bch[4 * v4 + 3]);
                  if (fullmap && bias)
                    bv = *reinterpret_cast<const float4*>(bias + pix % ((size_t)g.n1 * g.n2) * COUT + c0ch + 4 * v4);
                  sum.x = fmaxf(sum.x + bv.x, 0.f), sum.y = fmaxf(sum.y + bv.y, 0.f);
                  sum.z = fmaxf(sum.z + bv.z, 0.f), sum.w = fmaxf(sum.w + bv.w, 0.f);
                }
                *reinterpret_cast<float4*>(op) = sum;
              }
            }
          }
          named_bar(1 + grp, 128);
        }
      }
      tc_fence_before();
      if (lane == 0) mbar_arrive(&tempty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

static GeoT make_geo_t(int batch, int n1, int n2) {
  GeoT g;
  g.n1 = n1, g.n2 = n2;
  g.wseg = n2 < WSEG ? n2 : WSEG;
  g.P = conv_tf32_box_cols(n2);
  g.nrb = (n1 + R - 1) / R;
  g.ncs = (n2 + g.wseg - 1) / g.wseg;
  g.units = batch * g.nrb * g.ncs;
  return g;
}

size_t conv2_tf32_smem_bytes(int n2) {
  const int wseg = n2 < WSEG ? n2 : WSEG, P = wseg + 10;
  const size_t strip_alloc = ((size_t)(R + 10) * P * 128 + GUARD_ROWS * 128 + 1023) & ~(size_t)1023;
  return strip_alloc + WSTAGES * WBYTES + 2 * 4 * ECH * SPS * 4 + 1024;
}

int conv2_tf32_box_rows() { return R + 10; }
// strip pitch: n2 + 5 for one column segment (shared zero padding between rows, as conv2_tc_box_cols), else 74
int conv_tf32_box_cols(int n2) { return n2 <= WSEG ? n2 + 5 : WSEG + 10; }
int wgrad_box_cols(int n2) { return (n2 < WSEG ? n2 : WSEG) + 10; }

int convg_tf32_kblocks(int cin, int cout) { return (cin / 32) * 11 * ((11 + 128 / cout - 1) / (128 / cout)); }

template <int CIN, int COUT, int MODE>
static cudaError_t set_smem(int n2) {
  return cudaFuncSetAttribute(k_conv_tf32<CIN, COUT, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)conv2_tf32_smem_bytes(n2));
}

cudaError_t setup_conv2_tf32(int n2) {
  cudaError_t e;
  if ((e = set_smem<64, 32, EPI_BIAS_RELU>(n2)) != cudaSuccess) return e;
  if ((e = set_smem<32, 32, EPI_BIAS_RELU>(n2)) != cudaSuccess) return e;
  if ((e = set_smem<32, 64, EPI_BIAS_RELU>(n2)) != cudaSuccess) return e;
  return set_smem<64, 64, EPI_BIAS_RELU>(n2);
}


template <int CIN, int COUT, int MODE>
static cudaError_t launch(const CUtensorMap* tm, const void* wpack, const float* bias, int fullmap, const float* mask,
                          int batch, int n1, int n2, float* out, int num_sms, cudaStream_t st) {
  GeoT g = make_geo_t(batch, n1, n2);
  const int grid = g.units < num_sms ? g.units : num_sms;
  k_conv_tf32<CIN, COUT, MODE><<<grid, 384, conv2_tf32_smem_bytes(n2), st>>>(
      *tm, reinterpret_cast<const float*>(wpack), bias, fullmap, mask, g, out);
  return cudaGetLastError();
}

cudaError_t launch_conv2_tf32(const CUtensorMap* tmH1, const void* wpack, const float* bias, int fullmap, int batch,
                              int n1, int n2, float* h2, int num_sms, cudaStream_t st) {
  return launch<64, 32, EPI_BIAS_RELU>(tmH1, wpack, bias, fullmap, nullptr, batch, n1, n2, h2, num_sms, st);
}

cudaError_t launch_convg_tf32(int cin, int cout, const CUtensorMap* tmIn, const void* wpack, const float* bias,
                              int batch, int n1, int n2, float* out, int num_sms, cudaStream_t st) {
  if (cin == 64 && cout == 32) return launch<64, 32, EPI_BIAS_RELU>(tmIn, wpack, bias, 0, nullptr, batch, n1, n2, out, num_sms, st);
  if (cin == 32 && cout == 32) return launch<32, 32, EPI_BIAS_RELU>(tmIn, wpack, bias, 0, nullptr, batch, n1, n2, out, num_sms, st);
  if (cin == 32 && cout == 64) return launch<32, 64, EPI_BIAS_RELU>(tmIn, wpack, bias, 0, nullptr, batch, n1, n2, out, num_sms, st);
  if (cin == 64 && cout == 64) return launch<64, 64, EPI_BIAS_RELU>(tmIn, wpack, bias, 0, nullptr, batch, n1, n2, out, num_sms, st);
  return cudaErrorInvalidValue;
}

DI_DEBUG_BINDER(di_debug_bind_k_conv2_tf32)

}  // namespace di
