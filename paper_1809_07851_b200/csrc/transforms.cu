// NK1 kernel transform, NK2 input transform, NK4 output transform (+ crop).
//
// Separable 2-D transforms of one t x t tile (Eq. 4):
//   Winograd      U = B^T d B,   V = G g G^T,   Y = A^T X A
//   Regular-FFT   U = DFT2(d) on the half spectrum k_w < h = t/2+1,
//                 V = conj(DFT2(pad_t(g))) / t^2 (cross-correlation, readings R5/R6),
//                 Y = first m x m of the unnormalised inverse real DFT (pruned)
//   Gauss-FFT     as Regular, but U stores (U_r+U_i, U_r, U_i), V stores
//                 (V_r, V_i-V_r, V_r+V_i) and the three real products
//                 are recombined in NK4: Re = T1-T3, Im = T1+T2.
//
// Layouts: n = (b*n_h + i)*n_w + j indexes tiles
// (P:962-965), e = k*h + l indexes transformed elements.
//   U [BN_pad/128][Z][K][128]   (blocked by 128 tiles, fc_u_off; n contiguous within a block)
//   V [Z][M][Kp]       (K-major: the A operand of the contraction; Kp = K rounded up to 4)
//   X [Z][M][BN_pad]
// Winograd: Z=E, M=C', K=C.  Regular: Z=E, M=2C', K=2C (real embedding
// [[V_r,-V_i],[V_i,V_r]] x [U_r;U_i]).  Gauss: Z=3E, M=C', K=C.
#include "common.h"

namespace {

// ---------------------------------------------------------------- NK1 ------
// One thread per (c', c) kernel; lanes run along c so the V stores coalesce.
__global__ void __launch_bounds__(256) nk1_kernel_transform(Geometry g, const ConvConsts *__restrict__ cc,
                                                            const float *__restrict__ w, float *__restrict__ V,
                                                            float *__restrict__ Vlo, int split) {
    __shared__ float s_cos[FC_MAX_T], s_sin[FC_MAX_T], s_G[64];
    const int t = g.t, r = g.r, h = g.h;
    for (int i = threadIdx.x; i < FC_MAX_T; i += blockDim.x) {
        s_cos[i] = cc->cosv[i];
        s_sin[i] = cc->sinv[i];
    }
    for (int i = threadIdx.x; i < 64; i += blockDim.x) s_G[i] = cc->G[i];
    __syncthreads();
    int co, c0, cstep;  // F16X3: one CTA per output channel c' (scale first), threads over c
    float sv = 1.f;
    if (split == 2) {
        co = blockIdx.x;
        sv = fc_row_vscale(g, w, co);
        c0 = blockIdx.y * blockDim.x + threadIdx.x;  // grid (C', channel blocks)
        cstep = gridDim.y * blockDim.x;
    } else {
        const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
        if (idx >= (long long)g.C * g.Cout) return;
        co = (int)(idx / g.C);
        c0 = (int)(idx % g.C);
        cstep = g.C;
    }
    const size_t zstride = (size_t)(g.cplx ? g.Cout : g.M) * g.Kp;
    // element range [e_lo, e_hi) (element-sharded plans; the whole E otherwise): z relative to
    // e_lo, plane groups of Er = e_hi - e_lo elements
    const int elo = g.e_lo, ehi = g.e_hi, Er = ehi - elo;
    for (int c = c0; c < g.C; c += cstep) {
    const float *ker = w + ((size_t)co * g.C + c) * r * r;
    auto store = [&](int z, int row, int col, float v) {
        fc_store_v(V, Vlo, (size_t)z * zstride + (size_t)row * g.Kp + col, v, split, sv);
    };
    if (g.method == CONV_WINOGRAD) {
        float T[8];
        for (int l = 0; l < t; ++l) {
            for (int p = 0; p < r; ++p) {  // T[p] = sum_q g[p][q] G[l][q]
                float a = 0.f;
                for (int q = 0; q < r; ++q) a = fmaf(ker[p * r + q], s_G[l * r + q], a);
                T[p] = a;
            }
            for (int k = 0; k < t; ++k) {  // V[k][l] = sum_p G[k][p] T[p]
                const int e = k * t + l;
                if (e < elo || e >= ehi) continue;
                float a = 0.f;
                for (int p = 0; p < r; ++p) a = fmaf(s_G[k * r + p], T[p], a);
                store(e - elo, co, c, a);
            }
        }
        continue;
    }
    // FFT: DFT2 of the implicitly zero-padded kernel, conj, / t^2
    const float inv = 1.0f / ((float)t * (float)t);
    float Tr[FC_MAX_T], Ti[FC_MAX_T];
    for (int l = 0; l < h; ++l) {
        for (int p = 0; p < r; ++p) {  // row DFT along q: sum_q g[p][q] e^{-2 pi i l q / t}
            float ar = 0.f, ai = 0.f;
            int ph = 0;
            for (int q = 0; q < r; ++q) {
                const float v = ker[p * r + q];
                ar = fmaf(v, s_cos[ph], ar);
                ai = fmaf(-v, s_sin[ph], ai);
                ph += l;
                if (ph >= t) ph -= t;
            }
            Tr[p] = ar;
            Ti[p] = ai;
        }
        for (int k = 0; k < t; ++k) {  // column DFT along p
            if (k * h + l < elo || k * h + l >= ehi) continue;
            float ar = 0.f, ai = 0.f;
            int ph = 0;
            for (int p = 0; p < r; ++p) {
                const float cs = s_cos[ph], sn = s_sin[ph];
                // (Tr + i Ti)(cos - i sin)
                ar = fmaf(Tr[p], cs, fmaf(Ti[p], sn, ar));
                ai = fmaf(Ti[p], cs, fmaf(-Tr[p], sn, ai));
                ph += k;
                if (ph >= t) ph -= t;
            }
            const float vr = ar * inv, vi = -ai * inv;  // conj(DFT) / t^2
            const int e = k * h + l - elo;
            if (g.method == CONV_REGULAR_FFT && g.cplx) {  // (V_r, V_i) planes
                store(2 * e, co, c, vr);
                store(2 * e + 1, co, c, vi);
            } else if (g.method == CONV_REGULAR_FFT) {  // real embedding [[V_r, -V_i], [V_i, V_r]]
                store(e, co, c, vr);
                store(e, co, g.C + c, -vi);
                store(e, g.Cout + co, c, vi);
                store(e, g.Cout + co, g.C + c, vr);
            } else {  // Gauss: V_r, V_i - V_r, V_r + V_i
                store(e, co, c, vr);
                store(Er + e, co, c, vi - vr);
                store(2 * Er + e, co, c, vr + vi);
            }
        }
    }
    }
}

// ---------------------------------------------------------------- NK2 ------
// CTA = (channel c, TN consecutive tiles).  Stage tiles in smem, row pass,
// column pass, write U with lanes along the tile index (coalesced).
__global__ void __launch_bounds__(256) nk2_input_transform(Geometry g, const ConvConsts *__restrict__ cc,
                                                           const float *__restrict__ in, float *__restrict__ U,
                                                           int TN) {
    extern __shared__ float smem[];
    const int t = g.t, m = g.m, h = g.h, E = g.E;
    const bool fft = g.method != CONV_WINOGRAD;
    float *s_tab = smem;                          // 2*FC_MAX_T (cos, sin) or 64 (BT)
    float *s_d = smem + 2 * FC_MAX_T;             // [TN][t][t]
    float *s_z = s_d + TN * t * t;                // [TN][t][h] (x2 for complex)
    for (int i = threadIdx.x; i < FC_MAX_T; i += blockDim.x) {
        if (fft) {
            s_tab[i] = cc->cosv[i];
            s_tab[FC_MAX_T + i] = cc->sinv[i];
        } else {
            s_tab[i] = cc->BT[i];
        }
    }
    const int c = blockIdx.y;
    const long long n0 = (long long)blockIdx.x * TN;
    const int tt = t * t;
    for (int idx = threadIdx.x; idx < TN * tt; idx += blockDim.x) {
        const int nn = idx / tt, rem = idx - nn * tt, a = rem / t, bb = rem - a * t;
        const long long n = n0 + nn;
        float v = 0.f;
        if (n < g.BN) {
            const int b = (int)(n / g.N), tile = (int)(n - (long long)b * g.N);
            const int ti = tile / g.n_w, tj = tile - ti * g.n_w;
            const int y = ti * m + a, x = tj * m + bb;
            if (y < g.H && x < g.W) v = __ldg(in + (((size_t)b * g.C + c) * g.H + y) * g.W + x);
        }
        s_d[idx] = v;
    }
    __syncthreads();
    const float *s_cos = s_tab, *s_sin = s_tab + FC_MAX_T, *s_BT = s_tab;
    // row pass along the W axis: Z[nn][a][l] = sum_b d[nn][a][b] R[l][b]
    const int hh = fft ? h : t;
    for (int idx = threadIdx.x; idx < TN * t * hh; idx += blockDim.x) {
        const int l = idx % hh, rest = idx / hh;  // rest = nn*t + a
        const float *drow = s_d + rest * t;
        if (fft) {
            float ar = 0.f, ai = 0.f;
            int ph = 0;
            for (int bb = 0; bb < t; ++bb) {
                const float v = drow[bb];
                ar = fmaf(v, s_cos[ph], ar);
                ai = fmaf(-v, s_sin[ph], ai);
                ph += l;
                if (ph >= t) ph -= t;
            }
            s_z[2 * idx] = ar;
            s_z[2 * idx + 1] = ai;
        } else {
            float a = 0.f;
            for (int bb = 0; bb < t; ++bb) a = fmaf(s_BT[l * t + bb], drow[bb], a);
            s_z[idx] = a;
        }
    }
    __syncthreads();
    // column pass along the H axis and store; nn fastest for coalescing.  F16X3: per-tile
    // max|U| in shared slots (s_d is free after the row pass), then per image in global
    unsigned int *s_tmax = reinterpret_cast<unsigned int *>(s_d);
    if (g.umax)
        for (int i = threadIdx.x; i < TN; i += blockDim.x) s_tmax[i] = 0u;
    __syncthreads();
    for (int idx = threadIdx.x; idx < TN * E; idx += blockDim.x) {
        const int nn = idx % TN, e = idx / TN;
        const long long n = n0 + nn;
        if (n >= g.BN) continue;
        const int k = e / hh, l = e - k * hh;
        if (fft) {
            float ar = 0.f, ai = 0.f;
            int ph = 0;
            const float *zc = s_z + 2 * ((size_t)nn * t * h + l);
            for (int a = 0; a < t; ++a) {
                const float zr = zc[2 * a * h], zi = zc[2 * a * h + 1];
                const float cs = s_cos[ph], sn = s_sin[ph];
                ar = fmaf(zr, cs, fmaf(zi, sn, ar));
                ai = fmaf(zi, cs, fmaf(-zr, sn, ai));
                ph += k;
                if (ph >= t) ph -= t;
            }
            if (g.method == CONV_REGULAR_FFT) {
                U[fc_u_off(g, n, c, e)] = ar;
                U[fc_u_off(g, n, g.C + c, e)] = ai;
            } else {
                U[fc_u_off(g, n, c, e)] = ar + ai;
                U[fc_u_off(g, n, c, E + e)] = ar;
                U[fc_u_off(g, n, c, 2 * E + e)] = ai;
            }
            if (g.umax) atomicMax(s_tmax + nn, __float_as_uint(fabsf(ar) + fabsf(ai)));
        } else {
            float a = 0.f;
            const float *zc = s_z + (size_t)nn * t * t + l;
            for (int aa = 0; aa < t; ++aa) a = fmaf(s_BT[k * t + aa], zc[aa * t], a);
            U[fc_u_off(g, n, c, e)] = a;
            if (g.umax) atomicMax(s_tmax + nn, __float_as_uint(fabsf(a)));
        }
    }
    if (g.umax) {
        __syncthreads();
        for (int i = threadIdx.x; i < TN; i += blockDim.x)
            if (n0 + i < g.BN && s_tmax[i]) atomicMax(g.umax + (n0 + i) / g.N, s_tmax[i]);
    }
}

// ---------------------------------------------------------------- NK4 ------
// CTA = (output channel c', TN consecutive tiles).  Load X (Gauss: combine
// T1-T3, T1+T2 on load), pruned inverse column pass (a < m), pruned inverse
// row pass (b < m), crop to Ho x Wo.
__global__ void __launch_bounds__(256) nk4_output_transform(Geometry g, const ConvConsts *__restrict__ cc,
                                                            const float *__restrict__ X, float *__restrict__ out,
                                                            int TN) {
    extern __shared__ float smem[];
    const int t = g.t, m = g.m, h = g.h, E = g.E;
    const bool fft = g.method != CONV_WINOGRAD;
    const int cw = fft ? 2 : 1;
    float *s_tab = smem;
    float *s_x = smem + 2 * FC_MAX_T;       // [TN][t][h] * cw
    float *s_z = s_x + TN * E * cw;         // [TN][m][h] * cw
    for (int i = threadIdx.x; i < FC_MAX_T; i += blockDim.x) {
        if (fft) {
            s_tab[i] = cc->cosv[i];
            s_tab[FC_MAX_T + i] = cc->sinv[i];
        } else {
            s_tab[i] = cc->AT[i];
        }
    }
    const int co = blockIdx.y;
    const long long n0 = (long long)blockIdx.x * TN;
    const size_t BNp = g.BN_pad, Mdim = g.Xm;
    for (int idx = threadIdx.x; idx < TN * E; idx += blockDim.x) {
        const int nn = idx % TN, e = idx / TN;
        const long long n = n0 + nn;
        float xr = 0.f, xi = 0.f;
        if (n < g.BN) {
            if (g.method == CONV_WINOGRAD) {
                xr = X[((size_t)e * Mdim + co) * BNp + n];
            } else if (g.method == CONV_REGULAR_FFT || g.gc) {  // Gauss combined by NK3: Regular layout
                xr = X[((size_t)e * Mdim + co) * BNp + n];
                xi = X[((size_t)e * Mdim + g.Cout + co) * BNp + n];
            } else {
                const float T1 = X[((size_t)e * Mdim + co) * BNp + n];
                const float T2 = X[((size_t)(E + e) * Mdim + co) * BNp + n];
                const float T3 = X[((size_t)(2 * E + e) * Mdim + co) * BNp + n];
                xr = T1 - T3;
                xi = T1 + T2;
            }
        }
        const size_t o = (size_t)nn * E + e;
        if (fft) {
            s_x[2 * o] = xr;
            s_x[2 * o + 1] = xi;
        } else {
            s_x[o] = xr;
        }
    }
    __syncthreads();
    const float *s_cos = s_tab, *s_sin = s_tab + FC_MAX_T, *s_AT = s_tab;
    const int hh = fft ? h : t;
    // column inverse: Z[nn][a][l] = sum_k Linv[a][k] X[nn][k][l], a < m
    for (int idx = threadIdx.x; idx < TN * m * hh; idx += blockDim.x) {
        const int l = idx % hh, rest = idx / hh, a = rest % m, nn = rest / m;
        if (fft) {
            float ar = 0.f, ai = 0.f;
            int ph = 0;
            const float *xc = s_x + 2 * ((size_t)nn * E + l);
            for (int k = 0; k < t; ++k) {
                const float xr = xc[2 * k * h], xi = xc[2 * k * h + 1];
                const float cs = s_cos[ph], sn = s_sin[ph];
                // (xr + i xi)(cos + i sin)
                ar = fmaf(xr, cs, fmaf(-xi, sn, ar));
                ai = fmaf(xr, sn, fmaf(xi, cs, ai));
                ph += a;
                if (ph >= t) ph -= t;
            }
            s_z[2 * idx] = ar;
            s_z[2 * idx + 1] = ai;
        } else {
            float acc = 0.f;
            const float *xc = s_x + (size_t)nn * E + l;
            for (int k = 0; k < t; ++k) acc = fmaf(s_AT[a * t + k], xc[k * t], acc);
            s_z[idx] = acc;
        }
    }
    __syncthreads();
    // row inverse (b < m) and crop; bb fastest, then tile, for coalesced stores
    for (int idx = threadIdx.x; idx < TN * m * m; idx += blockDim.x) {
        const int bb = idx % m, rest = idx / m, nn = rest % TN, a = rest / TN;
        const long long n = n0 + nn;
        if (n >= g.BN) continue;
        const int b = (int)(n / g.N), tile = (int)(n - (long long)b * g.N);
        const int ti = tile / g.n_w, tj = tile - ti * g.n_w;
        const int y = ti * m + a, x = tj * m + bb;
        if (y >= g.Ho || x >= g.Wo) continue;
        float acc;
        if (fft) {
            const float *zr = s_z + 2 * (((size_t)nn * m + a) * h);
            acc = zr[0];  // l = 0 bin (imaginary part ignored, reading R7)
            int ph = bb;
            for (int l = 1; l < h; ++l) {
                const float wgt = (2 * l == t) ? 1.f : 2.f;
                acc = fmaf(wgt, fmaf(zr[2 * l], s_cos[ph], -zr[2 * l + 1] * s_sin[ph]), acc);
                ph += bb;
                if (ph >= t) ph -= t;
            }
        } else {
            const float *zr = s_z + ((size_t)nn * m + a) * t;
            acc = 0.f;
            for (int l = 0; l < t; ++l) acc = fmaf(s_AT[bb * t + l], zr[l], acc);
        }
        out[(((size_t)b * g.Cout + co) * g.Ho + y) * g.Wo + x] = acc;
    }
}

int pick_tn(int t) {
    if (t <= 16) return 32;
    if (t <= 24) return 16;
    if (t <= 32) return 8;
    if (t <= 45) return 4;
    return 2;
}

}  // namespace

cudaError_t fc_launch_kernel_transform(const Geometry &g, const ConvConsts *dc, const float *w, float *V,
                                       float *Vlo, int split, cudaStream_t s) {
    const long long n = (long long)g.C * g.Cout;
    if (split == 2) {
        const int bs = g.C >= 256 ? 256 : (g.C + 31) / 32 * 32;
        nk1_kernel_transform<<<dim3((unsigned)g.Cout, (unsigned)((g.C + bs - 1) / bs)), bs, 0, s>>>(g, dc, w, V, Vlo,
                                                                                                  split);
    } else {
        nk1_kernel_transform<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(g, dc, w, V, Vlo, split);
    }
    return cudaGetLastError();
}

cudaError_t fc_launch_input_transform(const Geometry &g, const ConvConsts *dc, const float *in, float *U,
                                      cudaStream_t s) {
    const int TN = pick_tn(g.t);
    const bool fft = g.method != CONV_WINOGRAD;
    const size_t smem = sizeof(float) * (2 * FC_MAX_T + (size_t)TN * g.t * g.t +
                                         (size_t)TN * g.t * (fft ? 2 * g.h : g.t));
    fc_smem_attr((const void *)nk2_input_transform, 200 * 1024);
    dim3 grid((unsigned)((g.BN + TN - 1) / TN), (unsigned)g.C);
    nk2_input_transform<<<grid, 256, smem, s>>>(g, dc, in, U, TN);
    return cudaGetLastError();
}

cudaError_t fc_launch_output_transform(const Geometry &g, const ConvConsts *dc, const float *X, float *out,
                                       cudaStream_t s) {
    const int TN = pick_tn(g.t);
    const bool fft = g.method != CONV_WINOGRAD;
    const int cw = fft ? 2 : 1;
    const size_t smem = sizeof(float) * (2 * FC_MAX_T + (size_t)TN * g.E * cw +
                                         (size_t)TN * g.m * (fft ? g.h : g.t) * cw);
    fc_smem_attr((const void *)nk4_output_transform, 200 * 1024);
    dim3 grid((unsigned)((g.BN + TN - 1) / TN), (unsigned)g.Cout);
    nk4_output_transform<<<grid, 256, smem, s>>>(g, dc, X, out, TN);
    return cudaGetLastError();
}
