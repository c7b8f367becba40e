/*
 * oracle/conv_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 CPU direct convolution: the parity
 * oracle for every method of the B200 fast-convolution path.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this file's library.  It shares NO code, header, constant or helper
 * with paper_1809_07851_b200/ (the CUDA product path), and never includes it.
 *
 * What it computes (Eq. 5 "eq:forward"):
 *
 *     I'_{b,c'} = sum_{c=1..C} I_{b,c} (*) W_{c'c}
 *
 * with (*) read as the "valid" cross-correlation (reading R1: no
 * kernel flip, as in ConvNet practice) and the weight index order
 * W[c'][c][p][q] (reading R2, "W_{c'c}"):
 *
 *     O[b][c'][i][j] = sum_{c<C} sum_{p<r} sum_{q<r}
 *                      (double)I[b][c][i+p][j+q] * (double)W[c'][c][p][q]
 *
 * for 0 <= i < H-r+1, 0 <= j < W-r+1 ("valid" output).  Winograd
 * and FFT convolution reach exactly this value in exact arithmetic (P:268-324,
 * P:372-384), so the plain definition is the oracle for all of them.
 *
 * Each output is accumulated sequentially in (c, p, q) order.  The loop nest
 * puts (i, j) innermost so the compiler may vectorise across outputs; that
 * does not change the per-output summation order.  Parallelism is over
 * (b, c') planes only, so results are bit-deterministic for any thread count.
 *
 * Every fp32 x fp32 product is exact in fp64 (24+24 <= 53 bits); only the
 * running sum rounds.  tests/test_oracle.py pins this file against math.fsum
 * brute force, hand-computed cases, torch's fp64 conv2d and invariants.
 */
#include <stddef.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Returns 0 on success, -1 on invalid shape. O is [B][Cout][H-r+1][W-r+1]. */
int oracle_conv_fp64(const float *I, const float *Wt, double *O,
                     int B, int C, int Cout, int H, int W, int r)
{
    if (B < 1 || C < 1 || Cout < 1 || r < 1 || H < r || W < r) return -1;
    const int Ho = H - r + 1, Wo = W - r + 1;
    const long long planes = (long long)B * Cout;
#pragma omp parallel for schedule(dynamic, 1)
    for (long long bc = 0; bc < planes; ++bc) {
        const int b = (int)(bc / Cout), co = (int)(bc % Cout);
        double *o = O + (size_t)bc * Ho * Wo;
        memset(o, 0, sizeof(double) * (size_t)Ho * Wo);
        for (int c = 0; c < C; ++c) {
            const float *img = I + ((size_t)b * C + c) * (size_t)H * W;
            const float *ker = Wt + ((size_t)co * C + c) * (size_t)r * r;
            for (int p = 0; p < r; ++p)
                for (int q = 0; q < r; ++q) {
                    const double w = (double)ker[p * r + q];
                    for (int i = 0; i < Ho; ++i) {
                        const float *row = img + (size_t)(i + p) * W + q;
                        double *orow = o + (size_t)i * Wo;
                        for (int j = 0; j < Wo; ++j)
                            orow[j] += (double)row[j] * w;
                    }
                }
        }
    }
    return 0;
}

/* Same definition, evaluated only at ns sampled outputs.
 * idx holds ns quadruples (b, c', i, j); out[s] receives O[b][c'][i][j].
 * Returns 0, or -1 on invalid shape / out-of-range index. */
int oracle_conv_fp64_sampled(const float *I, const float *Wt,
                             const int64_t *idx, long long ns, double *out,
                             int B, int C, int Cout, int H, int W, int r)
{
    if (B < 1 || C < 1 || Cout < 1 || r < 1 || H < r || W < r) return -1;
    const int Ho = H - r + 1, Wo = W - r + 1;
    for (long long s = 0; s < ns; ++s) {
        const int64_t *q4 = idx + 4 * s;
        if (q4[0] < 0 || q4[0] >= B || q4[1] < 0 || q4[1] >= Cout ||
            q4[2] < 0 || q4[2] >= Ho || q4[3] < 0 || q4[3] >= Wo) return -1;
    }
#pragma omp parallel for schedule(static)
    for (long long s = 0; s < ns; ++s) {
        const int b = (int)idx[4 * s], co = (int)idx[4 * s + 1];
        const int i = (int)idx[4 * s + 2], j = (int)idx[4 * s + 3];
        double acc = 0.0;
        for (int c = 0; c < C; ++c) {
            const float *img = I + ((size_t)b * C + c) * (size_t)H * W;
            const float *ker = Wt + ((size_t)co * C + c) * (size_t)r * r;
            for (int p = 0; p < r; ++p)
                for (int q = 0; q < r; ++q)
                    acc += (double)img[(size_t)(i + p) * W + (j + q)] *
                           (double)ker[p * r + q];
        }
        out[s] = acc;
    }
    return 0;
}

/* N-dimensional, non-isotropic form of the same definition (PAPER.md P:926-929:
 * "Extension to non-isotropic and N-dimensional images and kernels ... is straightforward"):
 *
 *     O[b][c'][o_0]..[o_{nd-1}] = sum_{c<C} sum_{p_0<r_0} .. sum_{p_{nd-1}<r_{nd-1}}
 *                                 (double)I[b][c][o_0+p_0]..[o_{nd-1}+p_{nd-1}]
 *                                 * (double)W[c'][c][p_0]..[p_{nd-1}]
 *
 * for 0 <= o_d < in[d] - r[d] + 1, nd = 1..3, row-major tensors.  Each output is summed
 * sequentially in (c, p_0, .., p_{nd-1}) order; parallel over (b, c') only.
 * Returns 0, or -1 on an invalid shape. */
int oracle_conv_nd_fp64(const float *I, const float *Wt, double *O, int nd, int B, int C, int Cout,
                        const int *in, const int *r)
{
    if (nd < 1 || nd > 3 || B < 1 || C < 1 || Cout < 1) return -1;
    int n[3] = {1, 1, 1}, k[3] = {1, 1, 1}, o[3] = {1, 1, 1};
    for (int d = 0; d < nd; ++d) {
        if (in[d] < 1 || r[d] < 1 || in[d] < r[d]) return -1;
        n[3 - nd + d] = in[d];
        k[3 - nd + d] = r[d];
        o[3 - nd + d] = in[d] - r[d] + 1;
    }
    const size_t vin = (size_t)n[0] * n[1] * n[2], vout = (size_t)o[0] * o[1] * o[2];
    const size_t kv = (size_t)k[0] * k[1] * k[2];
    const long long planes = (long long)B * Cout;
#pragma omp parallel for schedule(dynamic, 1)
    for (long long bc = 0; bc < planes; ++bc) {
        const int b = (int)(bc / Cout), co = (int)(bc % Cout);
        double *out = O + (size_t)bc * vout;
        for (int i0 = 0; i0 < o[0]; ++i0)
            for (int i1 = 0; i1 < o[1]; ++i1)
                for (int i2 = 0; i2 < o[2]; ++i2) {
                    double acc = 0.0;
                    for (int c = 0; c < C; ++c) {
                        const float *img = I + ((size_t)b * C + c) * vin;
                        const float *ker = Wt + ((size_t)co * C + c) * kv;
                        for (int p0 = 0; p0 < k[0]; ++p0)
                            for (int p1 = 0; p1 < k[1]; ++p1)
                                for (int p2 = 0; p2 < k[2]; ++p2)
                                    acc += (double)img[((size_t)(i0 + p0) * n[1] + (i1 + p1)) * n[2] + (i2 + p2)] *
                                           (double)ker[((size_t)p0 * k[1] + p1) * k[2] + p2];
                    }
                    out[((size_t)i0 * o[1] + i1) * o[2] + i2] = acc;
                }
    }
    return 0;
}

/* Gradients of the same layer (the adjoints of Eq. 5, written out; not in the paper):
 *   dX[b][c][y][x]    = sum_{c'} sum_{p,q : 0 <= y-p < Ho, 0 <= x-q < Wo} dY[b][c'][y-p][x-q] W[c'][c][p][q]
 *   dW[c'][c][p][q]   = sum_b sum_{i<Ho} sum_{j<Wo} dY[b][c'][i][j] I[b][c][i+p][j+q]
 * fp64 accumulation in (c', p, q) / (b, i, j) order; parallel over output planes only. */
int oracle_conv_bwd_data_fp64(const float *dY, const float *Wt, double *dX, int B, int C, int Cout, int H, int W,
                              int r)
{
    if (B < 1 || C < 1 || Cout < 1 || r < 1 || H < r || W < r) return -1;
    const int Ho = H - r + 1, Wo = W - r + 1;
    const long long planes = (long long)B * C;
#pragma omp parallel for schedule(dynamic, 1)
    for (long long bc = 0; bc < planes; ++bc) {
        const int b = (int)(bc / C), c = (int)(bc % C);
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x) {
                double acc = 0.0;
                for (int co = 0; co < Cout; ++co)
                    for (int p = 0; p < r; ++p)
                        for (int q = 0; q < r; ++q) {
                            const int i = y - p, j = x - q;
                            if (i < 0 || i >= Ho || j < 0 || j >= Wo) continue;
                            acc += (double)dY[(((size_t)b * Cout + co) * Ho + i) * Wo + j] *
                                   (double)Wt[(((size_t)co * C + c) * r + p) * r + q];
                        }
                dX[(((size_t)b * C + c) * H + y) * W + x] = acc;
            }
    }
    return 0;
}

int oracle_conv_bwd_filter_fp64(const float *I, const float *dY, double *dW, int B, int C, int Cout, int H, int W,
                                int r)
{
    if (B < 1 || C < 1 || Cout < 1 || r < 1 || H < r || W < r) return -1;
    const int Ho = H - r + 1, Wo = W - r + 1;
    const long long planes = (long long)Cout * C;
#pragma omp parallel for schedule(dynamic, 1)
    for (long long cc = 0; cc < planes; ++cc) {
        const int co = (int)(cc / C), c = (int)(cc % C);
        for (int p = 0; p < r; ++p)
            for (int q = 0; q < r; ++q) {
                double acc = 0.0;
                for (int b = 0; b < B; ++b)
                    for (int i = 0; i < Ho; ++i)
                        for (int j = 0; j < Wo; ++j)
                            acc += (double)dY[(((size_t)b * Cout + co) * Ho + i) * Wo + j] *
                                   (double)I[(((size_t)b * C + c) * H + i + p) * W + j + q];
                dW[(((size_t)co * C + c) * r + p) * r + q] = acc;
            }
    }
    return 0;
}

/* Threads the OpenMP runtime will use (reported as cpu_baseline.cores). */
int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
