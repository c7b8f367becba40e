// Register-resident complex FFTs of compile-time size N (mixed radix,
// Cooley-Tukey decimation in time; prime factors by dense DFT) used by the
// FFT tile transforms.  The paper's CPU codelets come from FFTW's genfft and
// "support arbitrary sizes"; here every size is unrolled
// at compile time instead, so all indices and twiddle addresses are constants.
//
// Twiddles W_N^k = exp(2 pi i k / N) live in __constant__ memory, computed on the
// host in fp64 and rounded once to fp32 (reading R11); after unrolling
// each FFMA reads its twiddle straight from the constant bank.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <mutex>

namespace fct {

struct cf {
    float x, y;
};

constexpr int kTwiddleCount = 64 * 65 / 2 + 64;  // sum_{N<=64} N, with slack
__constant__ float2 c_tw[kTwiddleCount];         // (cos, sin)(2 pi k / N) at tw_base(N) + k

__host__ __device__ constexpr int tw_base(int N) { return N * (N - 1) / 2; }

// a * W_N^(DIR*j) with the trivial angles special-cased at compile time
template <int N, int DIR>
__device__ __forceinline__ cf twiddle_mul(cf a, int j) {
    j %= N;
    if (j == 0) return a;
    if (2 * j == N) return cf{-a.x, -a.y};
    if (4 * j == N) return DIR > 0 ? cf{-a.y, a.x} : cf{a.y, -a.x};        // * (+-i)
    if (4 * j == 3 * N) return DIR > 0 ? cf{a.y, -a.x} : cf{-a.y, a.x};    // * (-+i)
    const float2 w = c_tw[tw_base(N) + j];
    const float s = DIR > 0 ? w.y : -w.y;
    return cf{fmaf(a.x, w.x, -a.y * s), fmaf(a.x, s, a.y * w.x)};
}

__host__ __device__ constexpr int radix_of(int n) {
    if (n % 4 == 0 && n > 4) return 4;
    for (int p = 2; p * p <= n; ++p)
        if (n % p == 0) return p;
    return n;
}

// dense DFT for small / prime sizes: X[k] = sum_n x[n] W_N^(DIR n k)
template <int N, int DIR>
__device__ __forceinline__ void dft_small(cf *x) {
    if constexpr (N == 1) {
        return;
    } else if constexpr (N == 2) {
        const cf a = x[0], b = x[1];
        x[0] = cf{a.x + b.x, a.y + b.y};
        x[1] = cf{a.x - b.x, a.y - b.y};
    } else if constexpr (N == 4) {
        const cf a = x[0], b = x[1], c = x[2], d = x[3];
        const cf s0{a.x + c.x, a.y + c.y}, s1{a.x - c.x, a.y - c.y};
        const cf s2{b.x + d.x, b.y + d.y}, s3{b.x - d.x, b.y - d.y};
        // s3 * (DIR i)
        const cf r3 = DIR > 0 ? cf{-s3.y, s3.x} : cf{s3.y, -s3.x};
        x[0] = cf{s0.x + s2.x, s0.y + s2.y};
        x[2] = cf{s0.x - s2.x, s0.y - s2.y};
        x[1] = cf{s1.x + r3.x, s1.y + r3.y};
        x[3] = cf{s1.x - r3.x, s1.y - r3.y};
    } else {
        // odd prime N: pair x_k with x_{N-k} (a_k = sum, b_k = difference), so each output
        // pair (j, N-j) costs (N-1)/2 real-coefficient complex FMAs on a and on b:
        //   y_j, y_{N-j} = x_0 + sum_k cos(2 pi jk/N) a_k  +-  i DIR sum_k sin(2 pi jk/N) b_k
        // (about half the multiplies of the dense O(N^2) complex products)
        constexpr int Hh = (N - 1) / 2;
        cf a[Hh], b[Hh];
        cf y0 = x[0];
#pragma unroll
        for (int k = 1; k <= Hh; ++k) {
            a[k - 1] = cf{x[k].x + x[N - k].x, x[k].y + x[N - k].y};
            b[k - 1] = cf{x[k].x - x[N - k].x, x[k].y - x[N - k].y};
            y0.x += a[k - 1].x;
            y0.y += a[k - 1].y;
        }
        cf y[N];
        y[0] = y0;
#pragma unroll
        for (int j = 1; j <= Hh; ++j) {
            cf re = x[0], im{-0.f, -0.f};
#pragma unroll
            for (int k = 1; k <= Hh; ++k) {
                const float2 w = c_tw[tw_base(N) + (j * k) % N];  // (cos, sin)(2 pi jk / N)
                re.x = fmaf(w.x, a[k - 1].x, re.x);
                re.y = fmaf(w.x, a[k - 1].y, re.y);
                im.x = fmaf(w.y, b[k - 1].x, im.x);
                im.y = fmaf(w.y, b[k - 1].y, im.y);
            }
            const cf t = DIR > 0 ? cf{-im.y, im.x} : cf{im.y, -im.x};  // i * DIR * im
            y[j] = cf{re.x + t.x, re.y + t.y};
            y[N - j] = cf{re.x - t.x, re.y - t.y};
        }
#pragma unroll
        for (int k = 0; k < N; ++k) x[k] = y[k];
    }
}

// in-place FFT, natural order in and out
template <int N, int DIR>
__device__ __forceinline__ void fft(cf *x) {
    constexpr int P = radix_of(N);
    if constexpr (P == N) {
        dft_small<N, DIR>(x);
    } else {
        constexpr int Q = N / P;
        cf s[P][Q];
#pragma unroll
        for (int n1 = 0; n1 < P; ++n1)
#pragma unroll
            for (int n2 = 0; n2 < Q; ++n2) s[n1][n2] = x[P * n2 + n1];
#pragma unroll
        for (int n1 = 0; n1 < P; ++n1) fft<Q, DIR>(s[n1]);
#pragma unroll
        for (int n1 = 1; n1 < P; ++n1)
#pragma unroll
            for (int k1 = 1; k1 < Q; ++k1) s[n1][k1] = twiddle_mul<N, DIR>(s[n1][k1], n1 * k1);
#pragma unroll
        for (int k1 = 0; k1 < Q; ++k1) {
            cf t[P];
#pragma unroll
            for (int n1 = 0; n1 < P; ++n1) t[n1] = s[n1][k1];
            dft_small<P, DIR>(t);
#pragma unroll
            for (int k2 = 0; k2 < P; ++k2) x[k1 + Q * k2] = t[k2];
        }
    }
}

// Host: upload THIS translation unit's copy of c_tw (without -rdc every TU that includes
// this header has its own __constant__ table) to the current device, once per device
// (thread-safe).  Called at plan creation (fc_init_twiddles), never inside a capture.
static inline cudaError_t upload_twiddles() {
    static std::mutex mu;
    static unsigned long long done_mask = 0;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    if (dev < 64 && ((done_mask >> dev) & 1ull)) return cudaSuccess;
    static float2 tab[kTwiddleCount];
    for (int N = 1; N <= 64; ++N)
        for (int k = 0; k < N; ++k) {  // fp64, rounded once (reading R11)
            const double ang = 2.0 * 3.14159265358979323846 * (double)k / (double)N;
            tab[tw_base(N) + k] = make_float2((float)std::cos(ang), (float)std::sin(ang));
        }
    e = cudaMemcpyToSymbol(c_tw, tab, sizeof(tab));
    if (e == cudaSuccess && dev < 64) done_mask |= 1ull << dev;
    return e;
}

}  // namespace fct

// host: upload every transform translation unit's twiddle table to the current device
cudaError_t fc_init_twiddles();
