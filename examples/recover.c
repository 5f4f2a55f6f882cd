/* recover.c -- the C ABI (include/deepinverse.h) from plain C: no CUDA headers, host buffers only.
 *
 * Builds a 16x16 problem (M = 64, batch 4) with its own LCG weights and measurements, recovers x_hat through
 * di_recover_host in a BF16 context, and checks two properties the method fixes exactly:
 *   y = 0 -> x_hat = 0 (zero biases), and positive homogeneity x_hat(2y) = 2 x_hat(y), bitwise (scaling by 2 is
 *   exact in binary floating point and every step of the map is positively homogeneous with zero biases).
 * Exit status 0 on success.
 *
 *   gcc -std=c99 -O2 -I include examples/recover.c -L paper_1701_03891_b200 -ldeepinverse \
 *       -Wl,-rpath,$PWD/paper_1701_03891_b200 -lm -o recover_c && ./recover_c
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "deepinverse.h"

static unsigned long long lcg = 1701;
static float unif(void) { /* [-1, 1) */
  lcg = lcg * 6364136223846793005ull + 1442695040888963407ull;
  return (float)((lcg >> 40) & 0xffffff) / 8388608.0f - 1.0f;
}
static void fill(float* p, size_t n, float scale) {
  for (size_t i = 0; i < n; ++i) p[i] = scale * unif();
}

int main(void) {
  enum { N1 = 16, N2 = 16, N = N1 * N2, M = 64, B = 4 };
  float* phi = malloc(sizeof(float) * M * N);
  float* w1 = malloc(sizeof(float) * 64 * 121);
  float* w2 = malloc(sizeof(float) * 32 * 64 * 121);
  float* w3 = malloc(sizeof(float) * 32 * 121);
  /* bf16 y is given as raw 16-bit patterns; build it from fp32 values by truncation to keep this file C only */
  unsigned short* y = malloc(sizeof(unsigned short) * B * M);
  unsigned short* y2 = malloc(sizeof(unsigned short) * B * M);
  unsigned short* y0 = calloc(B * M, sizeof(unsigned short));
  float* x = malloc(sizeof(float) * B * N);
  float* x2 = malloc(sizeof(float) * B * N);
  float* xz = malloc(sizeof(float) * B * N);
  fill(phi, (size_t)M * N, 0.125f);
  fill(w1, 64 * 121, 0.15f);
  fill(w2, (size_t)32 * 64 * 121, 0.02f);
  fill(w3, 32 * 121, 0.03f);
  for (int i = 0; i < B * M; ++i) {
    float v = unif();
    unsigned int u;
    memcpy(&u, &v, 4);
    y[i] = (unsigned short)(u >> 16);
    float v2 = 2.0f * v; /* exactly representable: the bf16 of 2v is 2 x (the bf16 of v) under truncation */
    memcpy(&u, &v2, 4);
    y2[i] = (unsigned short)(u >> 16);
  }
  di_create_args a;
  memset(&a, 0, sizeof a);
  a.m = M, a.n1 = N1, a.n2 = N2, a.phi = phi, a.phi_dtype = DI_DTYPE_F32;
  a.w1 = w1, a.w2 = w2, a.w3 = w3; /* NULL biases: zero */
  a.precision = DI_PREC_BF16, a.flags = 0, a.device = 0, a.max_batch = B;
  di_ctx ctx = NULL;
  di_status s = di_create(&a, &ctx);
  if (s != DI_OK) {
    fprintf(stderr, "di_create: %s: %s\n", di_status_string(s), di_last_error());
    return 2;
  }
  if ((s = di_recover_host(ctx, y, M, B, x, NULL)) != DI_OK || (s = di_recover_host(ctx, y2, M, B, x2, NULL)) != DI_OK ||
      (s = di_recover_host(ctx, y0, M, B, xz, NULL)) != DI_OK) {
    fprintf(stderr, "di_recover_host: %s: %s\n", di_status_string(s), di_last_error());
    return 3;
  }
  int bad = 0;
  double norm = 0.0;
  for (int i = 0; i < B * N; ++i) {
    bad += (x2[i] != 2.0f * x[i]) + (xz[i] != 0.0f);
    norm += (double)x[i] * x[i];
  }
  /* argument errors are reported synchronously, before any work */
  const int arg_ok = di_recover_host(ctx, y, M - 1, B, x, NULL) == DI_ERR_DIM &&
                     di_recover_host(ctx, y, M, B + 1, x, NULL) == DI_ERR_ARG;
  di_destroy(ctx);
  printf("{\"images\": %d, \"norm\": %.6g, \"homogeneity_and_zero_mismatches\": %d, \"arg_errors_ok\": %d}\n", B,
         sqrt(norm), bad, arg_ok);
  free(phi), free(w1), free(w2), free(w3), free(y), free(y2), free(y0), free(x), free(x2), free(xz);
  return (bad == 0 && arg_ok && norm > 0.0) ? 0 : 1;
}
