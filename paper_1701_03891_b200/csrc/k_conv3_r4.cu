// k_conv3_r4.cu -- stage 3 of the bf16 path, conv layer 3 (1 filter 11x11x32 + bias, ReLU iff DI_FLAG_FINAL_RELU,
// crop S) with RP = 4 or 8 OUTPUT ROWS STACKED IN M (C3R_RP in kernels.cuh; 8 by default --
// the description below is for 4: with 8, M = 8 rows x 16 (11 column taps), 18 windows, stack entries of 16 rows).
//
// C_out = 1 leaves the UMMA M dimension to the taps.  The first design (k_conv3_tc) stacks the 11 column taps of one
// tap row in M = 32 (.ws) and walks the 11 tap rows as K-blocks, so every strip position is read by 11 MMAs per
// 246 outputs and the tensor core's shared-memory reads bound it (0.87 ms at lowrate).  Here M = 128 = RP output rows
// t x ES rows (11 column taps v, padded): window k (k = 0 .. RP + 9) is the strip shifted by k rows, and rows (t, .)
// of its A operand hold the taps of tap row u = k - t, so that
//   D[(t, v)][n] = sum_k sum_c W[k - t][v][c] strip[n + k P][c]  and  x_hat[row RP p + t][j] = sum_v D[(t, v)][j + v].
// A_k = [W[k]; W[k-1]; ...; W[k-RP+1]] is a 128-row window of ONE stack T[i] = W[10 - i] (zero outside 0..10): A_k
// starts at T[10 - k], the whole bank stays resident in shared memory, and a window is a descriptor start address.
// N = P rounded up to 16 (<= 80) covers one strip row.  RP = 8 (ES = 16): per 8 x 64 outputs 18 windows x 2 MMAs
// (K = 16) of 6.5 KB of operands -- 0.07 MMAs per output against 0.09 (k_conv3_tc) and 0.11 (RP = 4): 0.43 ms.
// Each epilogue warp owns RPW = 32 / ES output rows (its TMEM quadrant) and sums their 11 diagonals through a
// private shared-memory tile.  (Streaming the strip one row per window instead, with RP = 11, measured slower: the
// per-window barrier handshake bounds the single issuing thread.)
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "sm100.cuh"

namespace di {

namespace {
constexpr int RP = C3R_RP, ES = C3R_ES, NWIN = C3R_NWIN, IMIN = C3R_IMIN;
constexpr int R = 8;                   // output rows per unit
constexpr int NPASS = R / RP;
constexpr int NACC = 4;                // TMEM accumulator slots (128 columns each)
constexpr int TBLK = ES * 64;          // one T entry: ES rows (v) x 32 channels bf16, SWIZZLE_64B
constexpr int TBYTES = (C3R_NENT * TBLK + 1023) & ~1023;
constexpr int GUARD = 16;              // zero positions past the strip (windows read up to N - P past the box)
constexpr int SROW = 84;               // epilogue tile row stride (floats): 16-B rows
constexpr int RPW = 32 / ES;           // output rows per epilogue warp (its TMEM quadrant)
constexpr int SWARP = RPW * 11 * SROW; // per epilogue warp

struct GeoR4 {
  int n1, n2, wseg, P, N, nrb, ncs, units;
};
}  // namespace

__global__ void __launch_bounds__(256, 1)
    k_conv3_r4(const __grid_constant__ CUtensorMap tmH2, const uint8_t* __restrict__ tpack,
               const float* __restrict__ bias, int fullmap, int relu, GeoR4 g, float* __restrict__ xhat) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int P = g.P;
  const int strip_bytes = (R + 10) * P * 64;
  const int strip_alloc = (strip_bytes + GUARD * 64 + 1023) & ~1023;
  uint8_t* const tb = smem;                                   // T stack (1024-aligned)
  uint8_t* const strip0 = smem + TBYTES;                      // 2 strips (TBYTES = 34 KB, 1024-aligned)
  float* const S = reinterpret_cast<float*>(smem + TBYTES + 2 * strip_alloc);

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
  if (warp == 2) tmem_alloc<512>(&tslot), tmem_relinquish();
  for (int s = 0; s < 2; ++s)   // finite guard past each strip
    for (int i = threadIdx.x; i < GUARD * 64 / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(strip0 + s * strip_alloc + strip_bytes)[i] = make_uint4(0, 0, 0, 0);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const int per_img = g.nrb * g.ncs;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ producer: T once, strips per unit
      mbar_arrive_expect_tx(&wbar, TBYTES);
      bulk_load(tb, tpack, TBYTES, &wbar);
      int it = 0;
      for (int u = blockIdx.x; u < g.units; u += gridDim.x, ++it) {
        const int b = u / per_img, rem = u - b * per_img;
        const int r0 = (rem / g.ncs) * R, c0 = (rem % g.ncs) * g.wseg;
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
      const uint32_t idesc = idesc_f32acc(1, 128, g.N);
      const uint64_t adesc0 = smem_desc(smem_u32(tb), 16, 512, kSwizzle64B);
      const uint64_t bdesc0 = smem_desc(smem_u32(strip0), 16, 512, kSwizzle64B);
      const uint64_t rstep = (uint64_t)((P * 64) >> 4);       // one strip row
      int it = 0, pi = 0;
      for (int u = blockIdx.x; u < g.units; u += gridDim.x, ++it) {
        const int s = it & 1;
        mbar_wait(&sfull[s], (it >> 1) & 1);
        tc_fence_after();
        for (int p = 0; p < NPASS; ++p, ++pi) {
          const int a = pi % NACC;
          if (pi >= NACC) {
            mbar_wait(&acc_empty[a], ((pi / NACC) - 1) & 1);
            tc_fence_after();
          }
          const uint32_t d = tmem + a * 128;
          uint64_t bd = bdesc0 + (uint64_t)((s * strip_alloc) >> 4) + (uint64_t)(RP * p) * rstep;
#pragma unroll 2
          for (int k = 0; k < NWIN; ++k, bd += rstep) {
            const uint64_t ad = adesc0 + (uint64_t)(((10 - k - IMIN) * TBLK) >> 4);   // T[10 - k] ..
            umma_f16_ss(d, ad, bd, idesc, k != 0);
            umma_f16_ss(d, ad + 2, bd + 2, idesc, 1);                       // channels 16..31: +32 B
          }
          umma_commit(&acc_full[a]);
        }
        umma_commit(&sempty[s]);
      }
    }
  } else if (warp >= 4) {  // ------------------------------- epilogue: warp q = output rows RPW q .. RPW q + RPW - 1
    const int q = warp - 4;
    float* const Sq = S + q * SWARP;
    const float bsc = (!fullmap && bias) ? bias[0] : 0.f;
    int pi = 0;
    for (int u = blockIdx.x; u < g.units; u += gridDim.x) {
      const int b = u / per_img, rem = u - b * per_img;
      const int r0 = (rem / g.ncs) * R, c0 = (rem % g.ncs) * g.wseg;
      for (int p = 0; p < NPASS; ++p, ++pi) {
        const int a = pi % NACC;
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
        if ((lane % ES) < 11) {   // S row (lane / ES) * 11 + v: tap v of output row RPW q + lane / ES
          float4* dst = reinterpret_cast<float4*>(Sq + ((lane / ES) * 11 + lane % ES) * SROW);
#pragma unroll
          for (int j = 0; j < 20; ++j)
            dst[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                 __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
        }
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2 * RPW; ++h) {
          const int j = lane + 32 * (h & 1), tr = h >> 1;
          const int row = r0 + RP * p + RPW * q + tr;
          float acc = 0.f;
#pragma unroll
          for (int v = 0; v < 11; ++v) acc += Sq[(tr * 11 + v) * SROW + j + v];
          if (j < g.wseg && c0 + j < g.n2 && row < g.n1) {
            const size_t pix = ((size_t)b * g.n1 + row) * g.n2 + c0 + j;
            acc += (fullmap && bias) ? bias[pix % ((size_t)g.n1 * g.n2)] : bsc;
            if (relu) acc = fmaxf(acc, 0.f);
            xhat[pix] = acc;
          }
        }
        __syncwarp();
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

static GeoR4 make_geo_r4(int batch, int n1, int n2) {
  GeoR4 g;
  g.n1 = n1, g.n2 = n2;
  g.wseg = n2 < 64 ? n2 : 64;
  g.P = g.wseg + 10;
  g.N = (g.P + 15) & ~15;
  g.nrb = (n1 + R - 1) / R;
  g.ncs = (n2 + g.wseg - 1) / g.wseg;
  g.units = batch * g.nrb * g.ncs;
  return g;
}

static size_t smem_r4(int n2) {
  const int wseg = n2 < 64 ? n2 : 64, P = wseg + 10;
  const size_t strip_alloc = ((size_t)(R + 10) * P * 64 + GUARD * 64 + 1023) & ~(size_t)1023;
  return TBYTES + 2 * strip_alloc + 4 * SWARP * 4 + 1024;
}

int conv3_r4_box_rows() { return R + 10; }
int conv3_r4_tpack_bytes() { return TBYTES; }

cudaError_t setup_conv3_r4(int n2) {
  return cudaFuncSetAttribute(k_conv3_r4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_r4(n2));
}

cudaError_t launch_conv3_r4(const CUtensorMap* tmH2, const void* tpack, const float* bias, int fullmap, int relu,
                            float* xhat, int batch, int n1, int n2, int num_sms, cudaStream_t st) {
  GeoR4 g = make_geo_r4(batch, n1, n2);
  const int grid = g.units < num_sms ? g.units : num_sms;
  k_conv3_r4<<<grid, 256, smem_r4(n2), st>>>(*tmH2, reinterpret_cast<const uint8_t*>(tpack), bias, fullmap, relu, g,
                                            xhat);
  return cudaGetLastError();
}

}  // namespace di
