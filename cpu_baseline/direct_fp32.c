/*
 * cpu_baseline/direct_fp32.c -- BASELINE ONLY (timed beside the GPU path by bench.py).
 *
 * The "straightforward multithreaded CPU direct conv" of BASELINE.json's north_star:
 * fp32 arithmetic, OpenMP over (b, c') output planes, the output row innermost so
 * the compiler vectorises along j (-O3 -mavx2 -mfma), no blocking or packing
 * tricks.  Same problem statement as the product path (Eq. 5,
 * valid cross-correlation, W[c'][c][p][q]; readings R1-R3).  It is not
 * the parity oracle (oracle/ is fp64) and shares no code with either.
 */
#include <stddef.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* O [B][Cout][H-r+1][W-r+1] (fp32).  Returns 0, or -1 on an invalid shape. */
int cpu_direct_fp32(const float *I, const float *Wt, float *O, int B, int C, int Cout, int H, int W, int r)
{
    if (B < 1 || C < 1 || Cout < 1 || r < 1 || H < r || W < r) return -1;
    const int Ho = H - r + 1, Wo = W - r + 1;
    const long long planes = (long long)B * Cout;
#pragma omp parallel for schedule(static)
    for (long long pl = 0; pl < planes; ++pl) {
        const int b = (int)(pl / Cout), co = (int)(pl % Cout);
        float *o = O + (size_t)pl * Ho * Wo;
        memset(o, 0, sizeof(float) * (size_t)Ho * Wo);
        for (int c = 0; c < C; ++c) {
            const float *in = I + ((size_t)b * C + c) * H * W;
            const float *w = Wt + ((size_t)co * C + c) * r * r;
            for (int p = 0; p < r; ++p)
                for (int q = 0; q < r; ++q) {
                    const float wv = w[p * r + q];
                    for (int i = 0; i < Ho; ++i) {
                        const float *row = in + (size_t)(i + p) * W + q;
                        float *orow = o + (size_t)i * Wo;
#pragma omp simd
                        for (int j = 0; j < Wo; ++j) orow[j] += wv * row[j];
                    }
                }
        }
    }
    return 0;
}

int cpu_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
