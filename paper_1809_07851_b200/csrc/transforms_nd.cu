// N-dimensional and non-isotropic layers (conv_plan_nd): NK1 / NK2 / NK4 as separable
// per-axis transforms of one tile, and the direct check path.
//
// "Extension to non-isotropic and N-dimensional images and kernels ...
// is straightforward.  The benchmarked implementations ... support an arbitrary number of
// dimensions, as well as non-isotropic kernels."  The fast algorithms are separable
// (Eq. 4 nests the 1-D transform along each axis; the DFT likewise), so an N-D
// tile transform is one 1-D transform per axis:
//   Winograd      U = (B_0^T x B_1^T x ...) d,  V = (G_0 x G_1 x ...) g,  Y = (A_0^T x A_1^T x ...) X
//                 with F(m_d, r_d) per axis (t_d = m_d + r_d - 1 <= 8; r_d = 1: identity, t_d = m_d)
//   Regular-FFT   forward DFT along every axis, the last one real-to-complex onto the half
//                 spectrum t/2 + 1 (P:1062-1065 generalised); V = conj(DFT(pad g)) / prod t_d;
//                 Y = the first m_d outputs per axis of the unnormalised inverse (c2c on the
//                 leading axes, c2r last, self-conjugate bins' imaginary parts dropped: R7)
//   Gauss-FFT     as Regular with the three-plane storage of P:427-441
// The contraction NK3 is unchanged (the same batched GEMM over E = prod_d len_d elements),
// and so are the U / V / X layouts (common.h).  Tiles are indexed row-major over the axes,
// n = b N + ((i_0 n_1) + i_1) n_2 + i_2, elements e = ((k_0 len_1) + k_1) len_2 + k_2.
//
// These kernels are generic (runtime sizes, dense per-axis matrices / DFTs through shared
// memory): the compile-time codelets of transforms_fast.cu / fft_xforms.cuh serve the 2-D
// isotropic layers the paper benchmarks.
#include <math.h>

#include "common.h"

namespace {

constexpr int NDT = 256;  // threads per CTA

struct NdSmem {
    float BT[3][64], G[3][64], AT[3][64];
    float cs[3][FC_MAX_T], sn[3][FC_MAX_T];
};

__device__ void nd_load_consts(NdSmem *sm, const NdConsts *__restrict__ dc) {
    const float *src = reinterpret_cast<const float *>(dc);
    float *dst = reinterpret_cast<float *>(sm);
    for (int i = threadIdx.x; i < (int)(sizeof(NdConsts) / sizeof(float)); i += blockDim.x) dst[i] = src[i];
}

enum PassKind { P_MAT = 0, P_DFT_FWD = 1, P_DFT_INV = 2, P_C2R = 3 };

// One 1-D transform along slot `ax` for `ntile` tiles of complex data in shared memory.
// in: dims L[0..2] row-major per tile (vin = L0 L1 L2 elements); out: the same dims with
// L[ax] replaced by Lout.  Kinds:
//   P_MAT      out[k] = sum_j Mx[k Lin + j] in[j]            (real matrix, Winograd)
//   P_DFT_FWD  out[k] = sum_j in[j] e^{-2 pi i k j / t}       (k < Lout <= t; Lin <= t)
//   P_DFT_INV  out[k] = sum_j in[j] e^{+2 pi i k j / t}
//   P_C2R      out[k] = Re(in[0]) + sum_{0<j<Lin} w_j Re(in[j] e^{+2 pi i k j / t}),
//              w_j = 1 for the t/2 bin of an even t, else 2: the inverse real DFT of a
//              half spectrum with the self-conjugate bins' imaginary parts dropped
// Accumulation in fp32 FMA, j ascending (twiddle index (k j) mod t from the fp64 table).
__device__ void nd_pass(const float2 *in, float2 *out, int ntile, const int *L, int ax, int Lout, int kind,
                        const float *Mx, const float *cs, const float *sn, int t) {
    int Lo[3] = {L[0], L[1], L[2]};
    Lo[ax] = Lout;
    const int vin = L[0] * L[1] * L[2], vout = Lo[0] * Lo[1] * Lo[2];
    const int Lin = L[ax];
    const int sin_ax = ax == 2 ? 1 : (ax == 1 ? L[2] : L[1] * L[2]);
    for (int idx = threadIdx.x; idx < ntile * vout; idx += blockDim.x) {
        const int tl = idx / vout, o = idx - tl * vout;
        int ii[3];
        ii[2] = o % Lo[2];
        ii[1] = (o / Lo[2]) % Lo[1];
        ii[0] = o / (Lo[1] * Lo[2]);
        const int k = ii[ax];
        ii[ax] = 0;
        const float2 *src = in + (size_t)tl * vin + (ii[0] * L[1] + ii[1]) * L[2] + ii[2];
        float ar = 0.f, ai = 0.f;
        if (kind == P_MAT) {
            for (int j = 0; j < Lin; ++j) {
                const float2 v = src[j * sin_ax];
                const float mj = Mx[k * Lin + j];
                ar = fmaf(mj, v.x, ar);
                ai = fmaf(mj, v.y, ai);
            }
        } else if (kind == P_DFT_FWD || kind == P_DFT_INV) {
            const float sg = kind == P_DFT_FWD ? -1.f : 1.f;
            int ph = 0;
            for (int j = 0; j < Lin; ++j) {
                const float2 v = src[j * sin_ax];
                const float c = cs[ph], s_ = sg * sn[ph];
                ar = fmaf(v.x, c, fmaf(-v.y, s_, ar));  // (v.x + i v.y)(c + i s)
                ai = fmaf(v.x, s_, fmaf(v.y, c, ai));
                ph += k;
                if (ph >= t) ph -= t;
            }
        } else {  // P_C2R
            ar = src[0].x;
            int ph = k % t;
            for (int j = 1; j < Lin; ++j) {
                const float2 v = src[j * sin_ax];
                const float wj = (2 * j == t) ? 1.f : 2.f;
                const float re = (2 * j == t) ? v.x * cs[ph] : fmaf(v.x, cs[ph], -v.y * sn[ph]);
                ar = fmaf(wj, re, ar);
                ph += k;
                if (ph >= t) ph -= t;
            }
        }
        out[(size_t)tl * vout + o] = make_float2(ar, ai);
    }
}

// tile n -> image b and per-axis tile coordinates
__device__ __forceinline__ void nd_tile(const Geometry &g, long long n, int &b, int *ti) {
    b = (int)(n / g.N);
    int tile = (int)(n - (long long)b * g.N);
    ti[2] = tile % g.ax_n[2];
    tile /= g.ax_n[2];
    ti[1] = tile % g.ax_n[1];
    ti[0] = tile / g.ax_n[1];
}

// ---------------------------------------------------------------- NK2 ------
// CTA = (channel c, TN consecutive tiles).  t-box of each tile (zero outside the input) ->
// per-axis forward transforms, last axis first (FFT: r2c onto the half spectrum) -> U.
__global__ void __launch_bounds__(NDT) nd_input_transform(Geometry g, const NdConsts *__restrict__ dc,
                                                          const float *__restrict__ in, float *__restrict__ U,
                                                          int TN) {
    extern __shared__ __align__(16) uint8_t smem_nd[];
    NdSmem *cst = reinterpret_cast<NdSmem *>(smem_nd);
    const int vt = g.ax_t[0] * g.ax_t[1] * g.ax_t[2];
    float2 *bufA = reinterpret_cast<float2 *>(smem_nd + sizeof(NdSmem));
    float2 *bufB = bufA + (size_t)TN * vt;
    unsigned int *s_tmax = reinterpret_cast<unsigned int *>(bufB + (size_t)TN * vt);
    nd_load_consts(cst, dc);
    const bool fft = g.method != CONV_WINOGRAD;
    const int c = blockIdx.y;
    const long long n0 = (long long)blockIdx.x * TN;
    for (int i = threadIdx.x; i < TN; i += blockDim.x) s_tmax[i] = 0u;
    for (int idx = threadIdx.x; idx < TN * vt; idx += blockDim.x) {
        const int tl = idx / vt, o = idx - tl * vt;
        const long long n = n0 + tl;
        float v = 0.f;
        if (n < g.BN) {
            int b, ti[3], p[3];
            nd_tile(g, n, b, ti);
            p[2] = o % g.ax_t[2];
            p[1] = (o / g.ax_t[2]) % g.ax_t[1];
            p[0] = o / (g.ax_t[1] * g.ax_t[2]);
            const int y0 = ti[0] * g.ax_m[0] + p[0], y1 = ti[1] * g.ax_m[1] + p[1], y2 = ti[2] * g.ax_m[2] + p[2];
            if (y0 < g.ax_in[0] && y1 < g.ax_in[1] && y2 < g.ax_in[2])
                v = __ldg(in + ((size_t)b * g.C + c) * (size_t)g.vin +
                          ((size_t)y0 * g.ax_in[1] + y1) * g.ax_in[2] + y2);
        }
        bufA[idx] = make_float2(v, 0.f);
    }
    __syncthreads();
    int L[3] = {g.ax_t[0], g.ax_t[1], g.ax_t[2]};
    float2 *src = bufA, *dst = bufB;
    for (int ax = 2; ax >= 3 - g.nd; --ax) {
        const int Lout = g.ax_len[ax];
        if (fft)
            nd_pass(src, dst, TN, L, ax, Lout, P_DFT_FWD, nullptr, cst->cs[ax], cst->sn[ax], g.ax_t[ax]);
        else
            nd_pass(src, dst, TN, L, ax, Lout, P_MAT, cst->BT[ax], nullptr, nullptr, g.ax_t[ax]);
        L[ax] = Lout;
        __syncthreads();
        float2 *tmp = src;
        src = dst;
        dst = tmp;
    }
    const int E = g.E;
    for (int idx = threadIdx.x; idx < TN * E; idx += blockDim.x) {
        const int tl = idx / E, e = idx - tl * E;
        const long long n = n0 + tl;
        if (n >= g.BN) continue;
        const float2 v = src[(size_t)tl * E + e];
        float mx;
        if (g.method == CONV_REGULAR_FFT) {
            U[fc_u_off(g, n, c, e)] = v.x;
            U[fc_u_off(g, n, g.C + c, e)] = v.y;
            mx = fabsf(v.x) + fabsf(v.y);
        } else if (fft) {  // Gauss: (U_r + U_i, U_r, U_i)
            U[fc_u_off(g, n, c, e)] = v.x + v.y;
            U[fc_u_off(g, n, c, E + e)] = v.x;
            U[fc_u_off(g, n, c, 2 * E + e)] = v.y;
            mx = fabsf(v.x) + fabsf(v.y);
        } else {
            U[fc_u_off(g, n, c, e)] = v.x;
            mx = fabsf(v.x);
        }
        if (g.umax) atomicMax(s_tmax + tl, __float_as_uint(mx));
    }
    if (g.umax) {  // F16X3: per-image max|U_b| (the contraction's per-image scale)
        __syncthreads();
        for (int i = threadIdx.x; i < TN; i += blockDim.x)
            if (n0 + i < g.BN && s_tmax[i]) atomicMax(g.umax + (n0 + i) / g.N, s_tmax[i]);
    }
}

// ---------------------------------------------------------------- NK4 ------
// CTA = (output channel c', TN consecutive tiles).  X of each tile (Gauss: T1 - T3, T1 + T2
// on load) -> inverse transforms on the leading axes (pruned to m_d outputs), the last axis
// last (FFT: c2r) -> the tile's m-box, cropped to the output.
__global__ void __launch_bounds__(NDT) nd_output_transform(Geometry g, const NdConsts *__restrict__ dc,
                                                           const float *__restrict__ X, float *__restrict__ out,
                                                           int TN) {
    extern __shared__ __align__(16) uint8_t smem_nd[];
    NdSmem *cst = reinterpret_cast<NdSmem *>(smem_nd);
    const int vt = g.ax_t[0] * g.ax_t[1] * g.ax_t[2];
    float2 *bufA = reinterpret_cast<float2 *>(smem_nd + sizeof(NdSmem));
    float2 *bufB = bufA + (size_t)TN * vt;
    nd_load_consts(cst, dc);
    const bool fft = g.method != CONV_WINOGRAD;
    const int co = blockIdx.y;
    const long long n0 = (long long)blockIdx.x * TN;
    const int E = g.E;
    const size_t BNp = g.BN_pad, Mdim = g.Xm;
    for (int idx = threadIdx.x; idx < TN * E; idx += blockDim.x) {
        const int tl = idx / E, e = idx - tl * E;
        const long long n = n0 + tl;
        float xr = 0.f, xi = 0.f;
        if (n < g.BN) {
            if (!fft) {
                xr = X[((size_t)e * Mdim + co) * BNp + n];
            } else if (g.method == CONV_REGULAR_FFT || g.gc) {
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
        bufA[idx] = make_float2(xr, xi);
    }
    __syncthreads();
    int L[3] = {g.ax_len[0], g.ax_len[1], g.ax_len[2]};
    float2 *src = bufA, *dst = bufB;
    for (int ax = 3 - g.nd; ax <= 2; ++ax) {  // leading axes first, the (half-spectrum) last axis last
        const int Lout = g.ax_m[ax];
        if (!fft)
            nd_pass(src, dst, TN, L, ax, Lout, P_MAT, cst->AT[ax], nullptr, nullptr, g.ax_t[ax]);
        else
            nd_pass(src, dst, TN, L, ax, Lout, ax == 2 ? P_C2R : P_DFT_INV, nullptr, cst->cs[ax], cst->sn[ax],
                    g.ax_t[ax]);
        L[ax] = Lout;
        __syncthreads();
        float2 *tmp = src;
        src = dst;
        dst = tmp;
    }
    const int vm = g.ax_m[0] * g.ax_m[1] * g.ax_m[2];
    for (int idx = threadIdx.x; idx < TN * vm; idx += blockDim.x) {
        const int tl = idx / vm, o = idx - tl * vm;
        const long long n = n0 + tl;
        if (n >= g.BN) continue;
        int b, ti[3], a[3];
        nd_tile(g, n, b, ti);
        a[2] = o % g.ax_m[2];
        a[1] = (o / g.ax_m[2]) % g.ax_m[1];
        a[0] = o / (g.ax_m[1] * g.ax_m[2]);
        const int y0 = ti[0] * g.ax_m[0] + a[0], y1 = ti[1] * g.ax_m[1] + a[1], y2 = ti[2] * g.ax_m[2] + a[2];
        if (y0 < g.ax_o[0] && y1 < g.ax_o[1] && y2 < g.ax_o[2])
            out[((size_t)b * g.Cout + co) * (size_t)g.vout + ((size_t)y0 * g.ax_o[1] + y1) * g.ax_o[2] + y2] =
                src[(size_t)tl * vm + o].x;
    }
}

// ---------------------------------------------------------------- NK1 ------
// CTA = (output channel c', TN input channels): the r-box of each kernel -> per-axis
// forward transforms (last axis first; Winograd G_d, FFT DFT of the zero-padded kernel
// onto t_d / the half spectrum) -> V in the contraction's layout (conj / prod t_d for FFT).
__global__ void __launch_bounds__(NDT) nd_kernel_transform(Geometry g, const NdConsts *__restrict__ dc,
                                                           const float *__restrict__ w, float *__restrict__ V,
                                                           float *__restrict__ Vlo, int split, int TN) {
    extern __shared__ __align__(16) uint8_t smem_nd[];
    NdSmem *cst = reinterpret_cast<NdSmem *>(smem_nd);
    const int vt = g.ax_t[0] * g.ax_t[1] * g.ax_t[2];
    float2 *bufA = reinterpret_cast<float2 *>(smem_nd + sizeof(NdSmem));
    float2 *bufB = bufA + (size_t)TN * vt;
    nd_load_consts(cst, dc);
    const bool fft = g.method != CONV_WINOGRAD;
    const int co = blockIdx.x;
    const int c0 = blockIdx.y * TN;
    const int nk = min(TN, g.C - c0);
    const float sv = split == 2 ? fc_row_vscale(g, w, co) : 1.f;
    const int kv = g.kvol;
    for (int idx = threadIdx.x; idx < TN * kv; idx += blockDim.x) {
        const int tl = idx / kv, o = idx - tl * kv;
        const float v = tl < nk ? __ldg(w + ((size_t)co * g.C + c0 + tl) * kv + o) : 0.f;
        bufA[idx] = make_float2(v, 0.f);
    }
    __syncthreads();
    int L[3] = {g.ax_r[0], g.ax_r[1], g.ax_r[2]};
    float2 *src = bufA, *dst = bufB;
    for (int ax = 2; ax >= 3 - g.nd; --ax) {
        const int Lout = g.ax_len[ax];
        if (fft)
            nd_pass(src, dst, TN, L, ax, Lout, P_DFT_FWD, nullptr, cst->cs[ax], cst->sn[ax], g.ax_t[ax]);
        else
            nd_pass(src, dst, TN, L, ax, Lout, P_MAT, cst->G[ax], nullptr, nullptr, g.ax_t[ax]);
        L[ax] = Lout;
        __syncthreads();
        float2 *tmp = src;
        src = dst;
        dst = tmp;
    }
    const int E = g.E;
    const float inv = 1.0f / (float)vt;
    const size_t zstride = (size_t)(g.cplx ? g.Cout : g.M) * g.Kp;
    auto store = [&](int z, int row, int col, float v) {
        fc_store_v(V, Vlo, (size_t)z * zstride + (size_t)row * g.Kp + col, v, split, sv);
    };
    for (int idx = threadIdx.x; idx < nk * E; idx += blockDim.x) {
        const int tl = idx / E, e = idx - tl * E, c = c0 + tl;
        const float2 v = src[(size_t)tl * E + e];
        if (!fft) {
            store(e, co, c, v.x);
            continue;
        }
        const float vr = v.x * inv, vi = -v.y * inv;  // conj(DFT) / prod t_d
        if (g.method == CONV_REGULAR_FFT && g.cplx) {
            store(2 * e, co, c, vr);
            store(2 * e + 1, co, c, vi);
        } else if (g.method == CONV_REGULAR_FFT) {
            store(e, co, c, vr);
            store(e, co, g.C + c, -vi);
            store(e, g.Cout + co, c, vi);
            store(e, g.Cout + co, g.C + c, vr);
        } else {
            store(e, co, c, vr);
            store(E + e, co, c, vi - vr);
            store(2 * E + e, co, c, vr + vi);
        }
    }
}

// ------------------------------------------------------------- direct (NK5) ---
// One thread per output element: sum over c and the kernel box in (c, kernel index) order.
__global__ void __launch_bounds__(NDT) nd_direct(Geometry g, const float *__restrict__ in,
                                                 const float *__restrict__ w, float *__restrict__ out) {
    const long long total = (long long)g.B * g.Cout * g.vout;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long plane = idx / g.vout;
        const int o = (int)(idx - plane * g.vout);
        const int b = (int)(plane / g.Cout), co = (int)(plane - (long long)b * g.Cout);
        const int o2 = o % g.ax_o[2], o1 = (o / g.ax_o[2]) % g.ax_o[1], o0 = o / (g.ax_o[1] * g.ax_o[2]);
        float acc = 0.f;
        for (int c = 0; c < g.C; ++c) {
            const float *img = in + ((size_t)b * g.C + c) * (size_t)g.vin;
            const float *ker = w + ((size_t)co * g.C + c) * (size_t)g.kvol;
            for (int p0 = 0; p0 < g.ax_r[0]; ++p0)
                for (int p1 = 0; p1 < g.ax_r[1]; ++p1)
                    for (int p2 = 0; p2 < g.ax_r[2]; ++p2)
                        acc = fmaf(img[((size_t)(o0 + p0) * g.ax_in[1] + o1 + p1) * g.ax_in[2] + o2 + p2],
                                   ker[(p0 * g.ax_r[1] + p1) * g.ax_r[2] + p2], acc);
        }
        out[idx] = acc;
    }
}

size_t nd_smem(int TN, int vt) { return sizeof(NdSmem) + 2 * (size_t)TN * vt * sizeof(float2) + 4 * (size_t)TN + 16; }

int nd_pick_tn(int vt) {
    int TN = (int)((96 * 1024) / (2 * (size_t)vt * sizeof(float2)));
    TN = TN > 64 ? 64 : TN;
    return TN < 1 ? 1 : TN;
}

}  // namespace

cudaError_t fc_launch_nd_stage(const Geometry &g, const NdConsts *dc, int stage, const float *src, float *dst,
                               float *Vlo, int split, cudaStream_t s) {
    const int vt = g.ax_t[0] * g.ax_t[1] * g.ax_t[2];
    if ((size_t)vt * 2 * sizeof(float2) > 200 * 1024) return cudaErrorInvalidConfiguration;
    int TN = nd_pick_tn(vt);
    const size_t smem = nd_smem(TN, vt);
    if (stage == 0) {
        fc_smem_attr((const void *)nd_kernel_transform, 200 * 1024);
        dim3 grid((unsigned)g.Cout, (unsigned)((g.C + TN - 1) / TN));
        nd_kernel_transform<<<grid, NDT, smem, s>>>(g, dc, src, dst, Vlo, split, TN);
    } else if (stage == 1) {
        fc_smem_attr((const void *)nd_input_transform, 200 * 1024);
        dim3 grid((unsigned)((g.BN + TN - 1) / TN), (unsigned)g.C);
        nd_input_transform<<<grid, NDT, smem, s>>>(g, dc, src, dst, TN);
    } else if (stage == 3) {
        fc_smem_attr((const void *)nd_output_transform, 200 * 1024);
        dim3 grid((unsigned)((g.BN + TN - 1) / TN), (unsigned)g.Cout);
        nd_output_transform<<<grid, NDT, smem, s>>>(g, dc, src, dst, TN);
    } else {
        return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t fc_launch_nd_direct(const Geometry &g, const float *in, const float *w, float *out, cudaStream_t s) {
    const long long total = (long long)g.B * g.Cout * g.vout;
    long long blocks = (total + NDT - 1) / NDT;
    blocks = blocks > 148LL * 64 ? 148LL * 64 : blocks;
    nd_direct<<<(unsigned)(blocks > 0 ? blocks : 1), NDT, 0, s>>>(g, in, w, out);
    return cudaGetLastError();
}
