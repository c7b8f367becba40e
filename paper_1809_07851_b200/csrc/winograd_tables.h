// Exact-rational Winograd F(m, r) matrices as *constant expressions*, so the
// compile-time-t transform kernels see every B^T / A^T / G entry as a literal
// (zeros and +-1 fold away).  Same construction as fc_winograd_rational() in
// api.cu (Eq. 1; reading R8): points
// {0, 1, -1, 2, -2, 1/2, -1/2} truncated to t-1 plus infinity,
// A^T = V_m^T, G = V_r, B^T = V^-T, B^T row denominators moved into G.
// tests/test_abi_host.py checks the runtime matrices exactly; the GPU parity
// tests exercise these compile-time copies end to end.
#pragma once

namespace wtab {

struct Fr {
    long long n, d;
};

__host__ __device__ constexpr long long gabs(long long a) { return a < 0 ? -a : a; }
__host__ __device__ constexpr long long ggcd(long long a, long long b) {
    a = gabs(a);
    b = gabs(b);
    while (b) {
        const long long t = a % b;
        a = b;
        b = t;
    }
    return a ? a : 1;
}
__host__ __device__ constexpr Fr fr(long long n, long long d) {
    if (d < 0) {
        n = -n;
        d = -d;
    }
    const long long g = ggcd(n, d);
    return Fr{n / g, d / g};
}
__host__ __device__ constexpr Fr fsub(Fr a, Fr b) { return fr(a.n * b.d - b.n * a.d, a.d * b.d); }
__host__ __device__ constexpr Fr fmul(Fr a, Fr b) { return fr(a.n * b.n, a.d * b.d); }
__host__ __device__ constexpr Fr fdiv(Fr a, Fr b) { return fr(a.n * b.d, a.d * b.n); }

struct Tables {
    double AT[8][8];  // [m][t]
    double BT[8][8];  // [t][t]
    double G[8][8];   // [t][r]
};

__host__ __device__ constexpr Fr point(int i) {
    const Fr pts[7] = {{0, 1}, {1, 1}, {-1, 1}, {2, 1}, {-2, 1}, {1, 2}, {-1, 2}};
    return pts[i];
}

__host__ __device__ constexpr Fr fpow(Fr p, int e) {
    Fr r{1, 1};
    for (int i = 0; i < e; ++i) r = fmul(r, p);
    return r;
}

__host__ __device__ constexpr Tables make(int m, int r) {
    const int t = m + r - 1;
    Tables out{};
    Fr V[8][8] = {}, Inv[8][8] = {};
    for (int i = 0; i < t; ++i)
        for (int j = 0; j < t; ++j) {
            V[i][j] = i < t - 1 ? fpow(point(i), j) : Fr{j == t - 1 ? 1 : 0, 1};
            Inv[i][j] = Fr{i == j ? 1 : 0, 1};
        }
    for (int col = 0; col < t; ++col) {
        int piv = col;
        while (piv < t && V[piv][col].n == 0) ++piv;
        for (int j = 0; j < t; ++j) {
            Fr x = V[col][j];
            V[col][j] = V[piv][j];
            V[piv][j] = x;
            x = Inv[col][j];
            Inv[col][j] = Inv[piv][j];
            Inv[piv][j] = x;
        }
        const Fr d = V[col][col];
        for (int j = 0; j < t; ++j) {
            V[col][j] = fdiv(V[col][j], d);
            Inv[col][j] = fdiv(Inv[col][j], d);
        }
        for (int i = 0; i < t; ++i) {
            if (i == col || V[i][col].n == 0) continue;
            const Fr f = V[i][col];
            for (int j = 0; j < t; ++j) {
                V[i][j] = fsub(V[i][j], fmul(f, V[col][j]));
                Inv[i][j] = fsub(Inv[i][j], fmul(f, Inv[col][j]));
            }
        }
    }
    for (int i = 0; i < t; ++i) {
        Fr bt[8] = {}, gm[8] = {};
        long long L = 1;
        for (int j = 0; j < t; ++j) {
            bt[j] = Inv[j][i];
            L = L / ggcd(L, bt[j].d) * bt[j].d;
        }
        for (int j = 0; j < r; ++j) gm[j] = i < t - 1 ? fpow(point(i), j) : Fr{j == r - 1 ? 1 : 0, 1};
        for (int j = 0; j < t; ++j) {
            const Fr v = fmul(bt[j], Fr{L, 1});
            out.BT[i][j] = (double)v.n / (double)v.d;
        }
        for (int j = 0; j < r; ++j) {
            const Fr v = fdiv(gm[j], Fr{L, 1});
            out.G[i][j] = (double)v.n / (double)v.d;
        }
    }
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < t; ++j) {
            const Fr v = j < t - 1 ? fpow(point(j), i) : Fr{i == m - 1 ? 1 : 0, 1};
            out.AT[i][j] = (double)v.n / (double)v.d;
        }
    return out;
}

// acc + c * x for a compile-time coefficient c: after unrolling, c is a literal and
// the branches fold, so zero coefficients cost nothing and +-1 become an add / sub
// (fmaf(0, x, acc) itself cannot be dropped under IEEE rules: 0 * inf = NaN).
// Accumulators start at -0.f, the additive identity that folds (-0 + x == x for all x).
__device__ __forceinline__ float cfma(double c, float x, float acc) {
    if (c == 0.0) return acc;
    if (c == 1.0) return acc + x;
    if (c == -1.0) return acc - x;
    return fmaf((float)c, x, acc);
}

// B^T depends on t only (the point set); A^T on (m, t); G on (r, t).
template <int T>
struct BTab {
    static constexpr Tables tab = make(2, T - 1);
};
template <int M, int T>
struct ATab {
    static constexpr Tables tab = make(M, T - M + 1);
};
template <int T, int R>
struct GTab {
    static constexpr Tables tab = make(T - R + 1, R);
};

}  // namespace wtab
