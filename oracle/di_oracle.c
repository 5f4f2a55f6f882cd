/*
 * di_oracle.c -- plain, slow, fp64 CPU oracle for the DeepInverse recovery map
 *                x_hat = M(y, Omega)   (§4).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_1701_03891_b200/csrc) and the CUDA path never calls it.
 *
 * Every function is the paper's definition written out, in the paper's order:
 *   dio_measure     y = Phi x (the measurement model)        PAPER.md:27 (§1)
 *   dio_proxy       x_tilde = Phi^T y                        PAPER.md:121 (§4)
 *                   viewed as n1 x n2, row-major j = r*n2+c  PAPER.md:122 (§4); SURVEY.md §8(c) Q8
 *   dio_conv_layer  Eq. (1): (x_c)^k_ij = S(ReLU((W^k * x)_ij + (b^k)_ij))
 *                   PAPER.md:123-128 (§4, Eq. 1); layers 2/3 "developed in a
 *                   similar manner" with a sum over input channels
 *
 *   dio_forward     x_tilde -> layer 1 -> layer 2 -> layer 3
 *   dio_train_grad  MSE loss L(Omega) and dL/dOmega by reverse-mode differentiation of the literal forward
 *                   PAPER.md:136 (§4); pinned by central finite differences (tests/test_oracle_train.py)
 *
 * Readings: '*' is the true (flipped-kernel) 2-D
 * convolution with full output size (n1+k1-1) x (n2+k2-1), zero outside the
 * input; S is the centred crop by (k-1)/2 (Q3); the
 * bias is either the full map of Eq. (1) or one scalar per output channel
 * (Q5); the ReLU of layer 3 is optional (Q6).
 *
 * Accumulation: fp64, for each output element the terms are added in the
 * order (c, u, v) ascending.
 */
#include <stdlib.h>
#include <string.h>

#define DIO_OK 0
#define DIO_ERR_ARG 1
#define DIO_ERR_DIM 2
#define DIO_ERR_OOM 5

/* y[b][i] = sum_j Phi[i][j] * x[b][j]   (y = Phi x, x vectorised row-major j = r*n2 + c).
 * phi: [m][n] row-major; x: [batch][n]; y: [batch][m]. */
int dio_measure(int m, int n, int batch, const double *phi, const double *x, double *y)
{
    if (m < 1 || n < 1 || batch < 0 || !phi || !x || !y) return DIO_ERR_ARG;
    for (int b = 0; b < batch; ++b) {
        const double *xb = x + (size_t)b * n;
        double *yb = y + (size_t)b * m;
        for (int i = 0; i < m; ++i) {
            double s = 0.0;
            for (int j = 0; j < n; ++j) s += phi[(size_t)i * n + j] * xb[j];
            yb[i] = s;
        }
    }
    return DIO_OK;
}

/* x_tilde[b][j] = sum_i Phi[i][j] * y[b][i]   (x_tilde = Phi^T y).
 * phi: [m][n] row-major; y: [batch][m]; xt: [batch][n]. */
int dio_proxy(int m, int n, int batch, const double *phi, const double *y, double *xt)
{
    if (m < 1 || n < 1 || batch < 0 || !phi || !y || !xt) return DIO_ERR_ARG;
    for (int b = 0; b < batch; ++b) {
        const double *yb = y + (size_t)b * m;
        double *xb = xt + (size_t)b * n;
        for (int j = 0; j < n; ++j) {
            double s = 0.0;
            for (int i = 0; i < m; ++i) s += phi[(size_t)i * n + j] * yb[i];
            xb[j] = s;
        }
    }
    return DIO_OK;
}

/* One convolutional layer, Eq. (1):
 *   F[o][i][j] = sum_c sum_u sum_v W[o][c][u][v] * X[c][i-u][j-v]  (X = 0 outside),
 *                0 <= i < n1+k-1, 0 <= j < n2+k-1            (full size)
 *   G = F + b            (full map b[o][i][j], or scalar b[o])
 *   H = ReLU(G) if relu
 *   Y[o][r][s] = H[o][r+p][s+p], p = (k-1)/2                 (S)
 * X: [cin][n1][n2]; W: [cout][cin][k][k]; Y: [cout][n1][n2].
 * xcorr != 0: the taps T are given in cross-correlation convention, i.e. the
 * filter of Eq. (1) is W[u][v] = T[k-1-u][k-1-v] (reading Q2). */
int dio_conv_layer(int cin, int cout, int n1, int n2, int k,
                   const double *X, const double *W, const double *bias, int fullmap_bias,
                   int relu, int xcorr, double *Y)
{
    if (cin < 1 || cout < 1 || n1 < 1 || n2 < 1 || k < 1 || (k % 2) == 0) return DIO_ERR_DIM;
    if (!X || !W || !Y) return DIO_ERR_ARG;
    const int h = n1 + k - 1, w = n2 + k - 1, p = (k - 1) / 2;
    double *F = (double *)malloc((size_t)h * w * sizeof(double));
    if (!F) return DIO_ERR_OOM;
    for (int o = 0; o < cout; ++o) {
        memset(F, 0, (size_t)h * w * sizeof(double));
        for (int c = 0; c < cin; ++c) {
            const double *Xc = X + (size_t)c * n1 * n2;
            for (int u = 0; u < k; ++u) {
                for (int v = 0; v < k; ++v) {
                    const int uu = xcorr ? k - 1 - u : u, vv = xcorr ? k - 1 - v : v;
                    const double wt = W[(((size_t)o * cin + c) * k + uu) * k + vv];
                    /* F[i][j] += W[u][v] * X[i-u][j-v] for the (i, j) where X is inside */
                    for (int i = u; i < u + n1; ++i) {
                        const double *xr = Xc + (size_t)(i - u) * n2;  /* X row i-u */
                        double *fr = F + (size_t)i * w + v;           /* F[i][v..]  */
                        for (int jj = 0; jj < n2; ++jj) fr[jj] += wt * xr[jj]; /* j = v + jj */
                    }
                }
            }
        }
        double *Yo = Y + (size_t)o * n1 * n2;
        for (int r = 0; r < n1; ++r)
            for (int s = 0; s < n2; ++s) {
                const int i = r + p, j = s + p;
                double g = F[(size_t)i * w + j];
                if (bias) g += fullmap_bias ? bias[((size_t)o * h + i) * w + j] : bias[o];
                if (relu && !(g > 0.0)) g = 0.0;
                Yo[(size_t)r * n2 + s] = g;
            }
    }
    free(F);
    return DIO_OK;
}

/* x_hat = M(y, Omega) for `batch` images, OpenMP over images only.
 * widths[0..nl]: channels (1, 64, 32, 1 for the paper);
 * w_all / b_all: layers concatenated ([cout][cin][k][k] each; biases [cout] or
 * [cout][n1+k-1][n2+k-1] each, or b_all == NULL for zero biases).
 * Every layer applies ReLU except the last unless final_relu. */
int dio_forward(int batch, int m, int n1, int n2, int nl, const int *widths, int k,
                const double *phi, const double *y, const double *w_all, const double *b_all,
                int fullmap_bias, int final_relu, int xcorr, double *xhat, int threads)
{
    if (batch < 0 || m < 1 || n1 < 1 || n2 < 1 || nl < 1 || !widths || !phi || !y || !w_all || !xhat)
        return DIO_ERR_ARG;
    if (widths[0] != 1 || widths[nl] != 1) return DIO_ERR_DIM;
    if ((long long)m > (long long)n1 * n2) return 3; /* M <= N */
    const int n = n1 * n2, h = n1 + k - 1, w = n2 + k - 1;
    int cmax = 1;
    for (int l = 0; l <= nl; ++l) if (widths[l] > cmax) cmax = widths[l];
    size_t woff[64], boff[64];
    if (nl > 63) return DIO_ERR_ARG;
    woff[0] = boff[0] = 0;
    for (int l = 0; l < nl; ++l) {
        woff[l + 1] = woff[l] + (size_t)widths[l + 1] * widths[l] * k * k;
        boff[l + 1] = boff[l] + (size_t)widths[l + 1] * (fullmap_bias ? (size_t)h * w : 1);
    }
    int err = DIO_OK;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads > 0 ? threads : 1)
    for (int b = 0; b < batch; ++b) {
        double *a = (double *)malloc((size_t)cmax * n * sizeof(double));
        double *t = (double *)malloc((size_t)cmax * n * sizeof(double));
        int e = (a && t) ? DIO_OK : DIO_ERR_OOM;
        if (e == DIO_OK) e = dio_proxy(m, n, 1, phi, y + (size_t)b * m, a);
        for (int l = 0; l < nl && e == DIO_OK; ++l) {
            const int relu = (l < nl - 1) || final_relu;
            e = dio_conv_layer(widths[l], widths[l + 1], n1, n2, k, a, w_all + woff[l],
                               b_all ? b_all + boff[l] : NULL, fullmap_bias, relu, xcorr, t);
            double *s = a; a = t; t = s;
        }
        if (e == DIO_OK) memcpy(xhat + (size_t)b * n, a, (size_t)n * sizeof(double));
        if (e != DIO_OK) {
#pragma omp critical
            err = e;
        }
        free(a); free(t);
    }
    return err;
}

/* ---------------------------------------------------------------------------------------------------------
 * Training gradients: the MSE loss of PAPER.md:136,
 *     L(Omega) = scale * sum_b ||M(y_b, Omega) - x_b||^2        (scale = 1/l for the paper's mean over l images)
 * and its gradient with respect to every W_l[o][c][u][v] (true-convolution orientation of Eq. (1)) and per-channel
 * bias b_l[o], by reverse-mode differentiation of the literal forward map:
 *     G = F + b on the full (n1+k-1) x (n2+k-1) map, F = W * X (true convolution), Y = S(act(G)):
 *     dG = S^T(dY) (zero outside the centred window) masked by act'(G) (ReLU: G > 0, i.e. Y > 0),
 *     db[o] = sum dG[o],  dW[o][c][u][v] = sum_{i,j} dG[o][i][j] X[c][i-u][j-v],
 *     dX[c][i'][j'] = sum_o sum_{u,v} W[o][c][u][v] dG[o][i'+u][j'+v].
 * The lifting layer Phi^T is fixed, so no gradient flows into Phi.
 * grad_w: [sum_l cout*cin*k*k], grad_b: [sum_l cout] (same concatenation as dio_forward's w_all / b_all with
 * per-channel biases).  Per-image gradients are accumulated per thread (static schedule) and summed in thread
 * order: deterministic for a fixed thread count. */
static void conv_backward(int cin, int cout, int n1, int n2, int k, const double *X, const double *W,
                          const double *Y, int relu, const double *dY, double *dW, double *db, double *dX)
{
    const int p = (k - 1) / 2;
    const size_t nn = (size_t)n1 * n2;
    double *dG = (double *)malloc(cout * nn * sizeof(double));
    for (int o = 0; o < cout; ++o)
        for (size_t q = 0; q < nn; ++q) {
            double g = dY[o * nn + q];
            if (relu && !(Y[o * nn + q] > 0.0)) g = 0.0;
            dG[o * nn + q] = g;
            db[o] += g;
        }
    /* in window coordinates (r, s) = (i - p, j - p): X[c][i-u][j-v] = X[c][r+p-u][s+p-v] */
    for (int o = 0; o < cout; ++o)
        for (int c = 0; c < cin; ++c)
            for (int u = 0; u < k; ++u)
                for (int v = 0; v < k; ++v) {
                    double acc = 0.0;
                    for (int r = 0; r < n1; ++r) {
                        const int xr = r + p - u;
                        if (xr < 0 || xr >= n1) continue;
                        for (int s = 0; s < n2; ++s) {
                            const int xs = s + p - v;
                            if (xs < 0 || xs >= n2) continue;
                            acc += dG[o * nn + (size_t)r * n2 + s] * X[c * nn + (size_t)xr * n2 + xs];
                        }
                    }
                    dW[(((size_t)o * cin + c) * k + u) * k + v] += acc;
                }
    if (dX) {
        memset(dX, 0, cin * nn * sizeof(double));
        for (int o = 0; o < cout; ++o)
            for (int c = 0; c < cin; ++c)
                for (int u = 0; u < k; ++u)
                    for (int v = 0; v < k; ++v) {
                        const double wt = W[(((size_t)o * cin + c) * k + u) * k + v];
                        for (int i = 0; i < n1; ++i) {            /* dX[c][i][j] += W dG[o][i+u-p][j+v-p] */
                            const int gr = i + u - p;
                            if (gr < 0 || gr >= n1) continue;
                            for (int j = 0; j < n2; ++j) {
                                const int gs = j + v - p;
                                if (gs < 0 || gs >= n2) continue;
                                dX[c * nn + (size_t)i * n2 + j] += wt * dG[o * nn + (size_t)gr * n2 + gs];
                            }
                        }
                    }
    }
    free(dG);
}

int dio_train_grad(int batch, int m, int n1, int n2, int nl, const int *widths, int k, const double *phi,
                   const double *y, const double *x_true, const double *w_all, const double *b_all, int final_relu,
                   double scale, double *grad_w, double *grad_b, double *loss, int threads)
{
    if (batch < 1 || m < 1 || n1 < 1 || n2 < 1 || nl < 1 || nl > 63 || !widths || !phi || !y || !x_true || !w_all ||
        !grad_w || !grad_b || !loss)
        return DIO_ERR_ARG;
    if (widths[0] != 1 || widths[nl] != 1 || (k % 2) == 0) return DIO_ERR_DIM;
    const size_t nn = (size_t)n1 * n2;
    size_t woff[64], boff[64];
    woff[0] = boff[0] = 0;
    int cmax = 1;
    for (int l = 0; l < nl; ++l) {
        woff[l + 1] = woff[l] + (size_t)widths[l + 1] * widths[l] * k * k;
        boff[l + 1] = boff[l] + (size_t)widths[l + 1];
        if (widths[l + 1] > cmax) cmax = widths[l + 1];
    }
    const size_t nw = woff[nl], nb = boff[nl];
    const int nt = threads > 0 ? threads : 1;
    double *acc = (double *)calloc((size_t)nt * (nw + nb + 1), sizeof(double));
    if (!acc) return DIO_ERR_OOM;
    int err = DIO_OK;
#pragma omp parallel num_threads(nt)
    {
#ifdef _OPENMP
        extern int omp_get_thread_num(void);
        const int tid = omp_get_thread_num();
#else
        const int tid = 0;
#endif
        double *gw = acc + (size_t)tid * (nw + nb + 1), *gb = gw + nw, *gl = gb + nb;
        double **act = (double **)calloc(nl + 1, sizeof(double *));
        double *dA = (double *)malloc(cmax * nn * sizeof(double)), *dB = (double *)malloc(cmax * nn * sizeof(double));
        int e = (act && dA && dB) ? DIO_OK : DIO_ERR_OOM;
        for (int l = 0; l <= nl && e == DIO_OK; ++l) {
            act[l] = (double *)malloc((size_t)widths[l] * nn * sizeof(double));
            if (!act[l]) e = DIO_ERR_OOM;
        }
#pragma omp for schedule(static)
        for (int b = 0; b < batch; ++b) {
            if (e != DIO_OK) continue;
            /* forward, keeping every layer's output */
            e = dio_proxy(m, (int)nn, 1, phi, y + (size_t)b * m, act[0]);
            for (int l = 0; l < nl && e == DIO_OK; ++l)
                e = dio_conv_layer(widths[l], widths[l + 1], n1, n2, k, act[l], w_all + woff[l],
                                   b_all ? b_all + boff[l] : NULL, 0, (l < nl - 1) || final_relu, 0, act[l + 1]);
            if (e != DIO_OK) continue;
            /* loss and dL/dx_hat = 2 scale (x_hat - x) */
            for (size_t q = 0; q < nn; ++q) {
                const double d = act[nl][q] - x_true[(size_t)b * nn + q];
                *gl += scale * d * d;
                dA[q] = 2.0 * scale * d;
            }
            /* backward through the conv layers; the fixed lifting layer gets no gradient */
            for (int l = nl - 1; l >= 0; --l) {
                conv_backward(widths[l], widths[l + 1], n1, n2, k, act[l], w_all + woff[l], act[l + 1],
                              (l < nl - 1) || final_relu, dA, gw + woff[l], gb + boff[l], l > 0 ? dB : NULL);
                double *t = dA; dA = dB; dB = t;
            }
        }
        if (e != DIO_OK) {
#pragma omp critical
            err = e;
        }
        for (int l = 0; l <= nl; ++l) free(act ? act[l] : NULL);
        free(act); free(dA); free(dB);
    }
    if (err == DIO_OK) {
        memset(grad_w, 0, nw * sizeof(double));
        memset(grad_b, 0, nb * sizeof(double));
        *loss = 0.0;
        for (int t = 0; t < nt; ++t) {                 /* fixed summation order */
            const double *gw = acc + (size_t)t * (nw + nb + 1);
            for (size_t i = 0; i < nw; ++i) grad_w[i] += gw[i];
            for (size_t i = 0; i < nb; ++i) grad_b[i] += gw[nw + i];
            *loss += gw[nw + nb];
        }
    }
    free(acc);
    return err;
}
