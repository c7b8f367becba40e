// FFT NK2 (input transform) and NK4 (inverse transform + crop) kernels, templated on the
// compile-time tile edge t; instantiated by fft_xforms_{a,b,c}.cu (split for parallel builds).
// Product path only.
#pragma once

#include "common.h"
#include "fft_tile.cuh"
#include "xform_util.cuh"

namespace fcfft {

using fct::cf;
using namespace fcx;

// ---------------------------------------------------------------- FFT NK2 ---
constexpr int FTN = 32;  // tiles per CTA (16 for grids of few CTAs, see launch_fft)

template <int T>
struct FftCfg {
    static constexpr int H = T / 2 + 1;
    static constexpr int S2 = (T * H) % 2 ? T * H : T * H + 1;  // odd stride (float2 units)
};

template <int T, int FT = FTN>
// flags: bit 0 channel-fastest grid, bit 1 tile rows 8-byte aligned (even W and m, aligned
// input): float2 row loads, half the L1 requests of the lanes' scattered 4-byte loads.
// 48 registers (5 CTAs/SM) for the composite t <= 16 codelets -- the kernel waits on its
// loads, more resident warps help (VGG-3.2 t = 10 NK2 172 -> 144 us, t = 16 119 -> 112 us);
// the prime-length DFTs (t = 11, 13) keep 64 (t = 13 measured 51 -> 64 us at 48)
__global__ void __launch_bounds__(256, ((T <= 16 && T % 2 == 0) || T == 9) ? 5 : ((T <= 18) ? 4 : 0)) nk2_fft(Geometry g, const float *__restrict__ in, float *__restrict__ U,
                                                                 int flags) {
    constexpr int H = FftCfg<T>::H, S = FftCfg<T>::S2, RP = (T + 1) / 2;
    extern __shared__ float2 zs[];  // [FT][S]: tile nn, row a, bin l at nn*S + a*H + l
    const int cfast = flags & 1;
    const int c = cfast ? blockIdx.x : blockIdx.y;
    const long long n0 = (long long)(cfast ? blockIdx.y : blockIdx.x) * FT;
    for (int it = threadIdx.x; it < RP * FT; it += blockDim.x) {
        const int nn = it % FT, p = it / FT;
        const int a0 = 2 * p, a1 = 2 * p + 1;
        const long long n = n0 + nn;
        cf z[T];
        if (n < g.BN) {
            const int b = fc_div((int)n, g.divN), tile = (int)n - b * g.N;
            const int ti = fc_div(tile, g.divNw), tj = tile - ti * g.n_w;
            const int y0 = ti * g.m, x0 = tj * g.m;
            const float *src = in + ((size_t)b * g.C + c) * g.H * g.W;
            const bool r0 = y0 + a0 < g.H, r1 = (a1 < T) && (y0 + a1 < g.H);
            const float *row0 = src + (size_t)(y0 + a0) * g.W + x0;
            const float *row1 = row0 + g.W;
            if (T % 2 == 0 && (flags & 2) && x0 + T <= g.W) {
#pragma unroll
                for (int q = 0; q < T; q += 2) {
                    const float2 u0 = r0 ? __ldg(reinterpret_cast<const float2 *>(row0 + q)) : make_float2(0.f, 0.f);
                    const float2 u1 = r1 ? __ldg(reinterpret_cast<const float2 *>(row1 + q)) : make_float2(0.f, 0.f);
                    z[q] = cf{u0.x, u1.x};
                    z[q + 1 < T ? q + 1 : q] = cf{u0.y, u1.y};
                }
            } else if (x0 + T <= g.W) {
#pragma unroll
                for (int q = 0; q < T; ++q) {
                    z[q].x = r0 ? __ldg(row0 + q) : 0.f;
                    z[q].y = r1 ? __ldg(row1 + q) : 0.f;
                }
            } else {
#pragma unroll
                for (int q = 0; q < T; ++q) {
                    const bool cx = x0 + q < g.W;
                    z[q].x = (r0 && cx) ? __ldg(row0 + q) : 0.f;
                    z[q].y = (r1 && cx) ? __ldg(row1 + q) : 0.f;
                }
            }
        } else {
#pragma unroll
            for (int q = 0; q < T; ++q) z[q] = cf{0.f, 0.f};
        }
        fct::fft<T, -1>(z);
        // split the spectra of the two real rows: Xa = (Z[l] + conj Z[-l]) / 2, Xb = (Z[l] - conj Z[-l]) / 2i
        float2 *dst = zs + nn * S + a0 * H;
#pragma unroll
        for (int l = 0; l < H; ++l) {
            const cf p_ = z[l], q_ = z[(T - l) % T];
            dst[l] = make_float2(0.5f * (p_.x + q_.x), 0.5f * (p_.y - q_.y));
            if (a1 < T) dst[H + l] = make_float2(0.5f * (p_.y + q_.y), -0.5f * (p_.x - q_.x));
        }
    }
    __syncthreads();
    float umx = 0.f;
    for (int it = threadIdx.x; it < H * FT; it += blockDim.x) {
        const int nn = it % FT, l = it / FT;
        const long long n = n0 + nn;
        cf z[T];
#pragma unroll
        for (int a = 0; a < T; ++a) {
            const float2 v = zs[nn * S + a * H + l];
            z[a] = cf{v.x, v.y};
        }
        fct::fft<T, -1>(z);
        if (n >= g.BN) continue;
#pragma unroll
        for (int k = 0; k < T; ++k) umx = fmaxf(umx, fabsf(z[k].x) + fabsf(z[k].y));
        // element e = k H + l at + e * zs: step the pointers by an opaque byte stride
        size_t hb = (size_t)H * fc_u_zs(g) * sizeof(float);
        asm("" : "+l"(hb));
        if (g.method == CONV_REGULAR_FFT) {  // rows c (Re) and C + c (Im)
            char *d0 = reinterpret_cast<char *>(U + fc_u_off(g, n, c, l));
            char *d1 = reinterpret_cast<char *>(U + fc_u_off(g, n, g.C + c, l));
#pragma unroll
            for (int k = 0; k < T; ++k) {
                *reinterpret_cast<float *>(d0) = z[k].x;
                *reinterpret_cast<float *>(d1) = z[k].y;
                d0 += hb;
                d1 += hb;
            }
        } else {  // Gauss: (U_r + U_i, U_r, U_i) in element planes 0, 1, 2 (z = plane * E + e)
            char *d0 = reinterpret_cast<char *>(U + fc_u_off(g, n, c, l));
            const size_t pl = (size_t)g.E * fc_u_zs(g) * sizeof(float);
#pragma unroll
            for (int k = 0; k < T; ++k) {
                *reinterpret_cast<float *>(d0) = z[k].x + z[k].y;
                *reinterpret_cast<float *>(d0 + pl) = z[k].x;
                *reinterpret_cast<float *>(d0 + 2 * pl) = z[k].y;
                d0 += hb;
            }
        }
    }
    if (g.umax) {  // per-image max|U|: a thread's items all have tile nn = threadIdx.x % FT
        const long long nt = n0 + (threadIdx.x % FT);
        fc_block_umax_img(g.umax, fc_div((int)(n0 < g.BN ? n0 : g.BN - 1), g.divN),
                          nt < g.BN ? fc_div((int)nt, g.divN) : -1, umx);
    }
}

// ---------------------------------------------------------------- FFT NK4 ---
// CTA = R tile rows of IPC consecutive images (their tiles are contiguous in n).
// Phase A: one (half-spectrum column l, tile) per thread -- load the t values of
// X along n (Gauss: T1-T3, T1+T2 on load), inverse FFT along the tile's H axis,
// keep the m output rows in shared memory.  Phase B: two output rows per complex
// inverse FFT (A + iB packing, self-conjugate bins' imaginary parts dropped,
// reading R7), cropped m x m block into a shared-memory output strip.  Phase C:
// coalesced streaming stores of each image's output rows.
template <int T>
__global__ void __launch_bounds__(512, (T <= 18) ? 2 : 0) nk4_fft(Geometry g, int R, int IPC, int SWo, const float *__restrict__ X,
                                               float *__restrict__ out) {
    constexpr int H = FftCfg<T>::H;
    const int m = g.m;
    const int S = (m * H) % 2 ? m * H : m * H + 1;
    const int strip = blockIdx.x, b = blockIdx.y * IPC, co = blockIdx.z;  // grid (strips, image groups, C')
    const int i0 = strip * R;
    const int ntr = min(R, g.n_h - i0);
    const int nimg = min(IPC, g.B - b);
    const int ntiles = nimg * ntr * g.n_w;
    const long long nbase = ((long long)b * g.n_h + i0) * g.n_w;
    extern __shared__ float2 zs[];                                     // [ntiles][S]
    float *so = reinterpret_cast<float *>(zs + (((size_t)IPC * R * g.n_w * S + 1) & ~(size_t)1));  // [nimg*ntr*m][SWo]
    const size_t estride = (size_t)g.Xm * g.BN_pad;
    // (stepping these loads by an opaque byte stride, as nk4_wino does, measured slower here:
    // VGG-1.2 t = 27 / 32 NK4 +7-9%, three-plane Gauss +13%)
    const size_t hstride = (size_t)H * estride;  // k -> k+1 along the element index e = k*H + l
    const float inv_nt = 1.f / (float)ntiles, inv_nw = 1.f / (float)g.n_w, inv_nh = 1.f / (float)g.n_h;
    // whole images of narrow rows (R = n_h, Wo < 48): phase B stages the cropped Ho x Wo planes
    // at pitch Wo and phase C copies each image out as one flat run (as nk4_wino)
    const bool whole = R == g.n_h && g.Wo < 48;
    for (int it = threadIdx.x; it < H * ntiles; it += blockDim.x) {
        const int l = fc_sdiv(it, inv_nt), tl = it - l * ntiles;
        cf z[T];
        const float *s0 = X + (size_t)co * g.BN_pad + nbase + tl + (size_t)l * estride;
        if (g.method == CONV_REGULAR_FFT || g.gc) {  // (Re, Im) rows c', C' + c' (Gauss: combined by NK3)
            const float *s1 = s0 + (size_t)g.Cout * g.BN_pad;
#pragma unroll
            for (int k = 0; k < T; ++k) z[k] = cf{__ldcs(s0 + k * hstride), __ldcs(s1 + k * hstride)};
        } else {  // Gauss: Re = T1 - T3, Im = T1 + T2
            const size_t pl = (size_t)g.E * estride;
#pragma unroll
            for (int k = 0; k < T; ++k) {
                const float *p = s0 + k * hstride;
                const float t1 = __ldcs(p), t2 = __ldcs(p + pl), t3 = __ldcs(p + 2 * pl);
                z[k] = cf{t1 - t3, t1 + t2};
            }
        }
        fct::fft<T, +1>(z);  // inverse along the tile's H axis (unnormalised; 1/t^2 sits in V)
        float2 *dst = zs + (size_t)tl * S + l;
#pragma unroll
        for (int a = 0; a < T; ++a)
            if (a < m) dst[a * H] = make_float2(z[a].x, z[a].y);
    }
    __syncthreads();
    const int RP = (m + 1) / 2;
    for (int it = threadIdx.x; it < RP * ntiles; it += blockDim.x) {
        const int p = fc_sdiv(it, inv_nt), tl = it - p * ntiles;
        const int a0 = 2 * p, a1 = 2 * p + 1;
        const float2 *ra = zs + (size_t)tl * S + a0 * H;
        const float2 *rb = ra + H;
        const bool has1 = a1 < m;
        cf z[T];
#pragma unroll
        for (int l = 0; l < H; ++l) {
            float2 A = ra[l];
            float2 Bv = has1 ? rb[l] : make_float2(0.f, 0.f);
            if (l == 0 || 2 * l == T) {  // self-conjugate bins: imaginary part dropped (reading R7)
                A.y = 0.f;
                Bv.y = 0.f;
            }
            z[l] = cf{A.x - Bv.y, A.y + Bv.x};                               // A + i B
            if (l > 0 && 2 * l < T) z[T - l] = cf{A.x + Bv.y, Bv.x - A.y};  // conj(A) + i conj(B)
        }
        fct::fft<T, +1>(z);
        const int ti = fc_sdiv(tl, inv_nw), tj = tl - ti * g.n_w;  // ti counts tile rows across the CTA's images
        if (whole) {  // cropped Ho x Wo planes back to back
            const int im = fc_sdiv(ti, inv_nh), oy = (ti - im * g.n_h) * m + a0, ox = tj * m;
            float *q = so + ((size_t)im * g.Ho + oy) * g.Wo + ox;
            const bool r0 = oy < g.Ho, r1 = has1 && oy + 1 < g.Ho;
#pragma unroll
            for (int c = 0; c < T; ++c)
                if (c < m && ox + c < g.Wo) {
                    if (r0) q[c] = z[c].x;
                    if (r1) q[g.Wo + c] = z[c].y;
                }
            continue;
        }
        float *q0 = so + (size_t)(ti * m + a0) * SWo + tj * m;
        if ((m & 1) == 0 && (SWo & 1) == 0) {  // 8-byte aligned pairs
#pragma unroll
            for (int q = 0; q + 1 < T; q += 2) {
                if (q < m) {
                    *reinterpret_cast<float2 *>(q0 + q) = make_float2(z[q].x, z[q + 1].x);
                    if (has1) *reinterpret_cast<float2 *>(q0 + SWo + q) = make_float2(z[q].y, z[q + 1].y);
                }
            }
        } else {
#pragma unroll
            for (int q = 0; q < T; ++q) {
                if (q < m) {
                    q0[q] = z[q].x;
                    if (has1) q0[SWo + q] = z[q].y;
                }
            }
        }
    }
    __syncthreads();
    if (whole) {  // every image's Ho x Wo plane is one contiguous run in both places
        const int plane = g.Ho * g.Wo;
        const bool vec = (plane & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
        const int n = vec ? plane >> 2 : plane;  // units (float4 or float) per image
        const size_t istride = (size_t)g.Cout * plane;
        float *dst0 = out + ((size_t)b * g.Cout + co) * plane;
        if (n >= (int)blockDim.x) {  // planes of at least one unit per thread: a loop per image
            float *dimg = dst0;
            for (int i = 0; i < nimg; ++i, dimg += istride) {
                if (vec)
                    for (int k = threadIdx.x; k < n; k += blockDim.x)
                        __stcs(reinterpret_cast<float4 *>(dimg) + k, reinterpret_cast<const float4 *>(so)[i * n + k]);
                else
                    for (int k = threadIdx.x; k < n; k += blockDim.x) __stcs(dimg + k, so[i * n + k]);
            }
            return;
        }
        // small planes: one flat (image, unit) walk over all images, the position advancing
        // by blockDim units per step with one division up front (a division per element was
        // ~25 instructions per float, ncu k5 m = 9 NK4; a loop per image costs every warp its
        // overhead per image: deep NK4 18 -> 25 us)
        const int q = (int)blockDim.x / n, rem = (int)blockDim.x - q * n;
        int im = (int)threadIdx.x / n, r = (int)threadIdx.x - im * n;
        while (im < nimg) {
            if (vec)
                __stcs(reinterpret_cast<float4 *>(dst0 + im * istride) + r,
                       reinterpret_cast<const float4 *>(so)[im * n + r]);
            else
                __stcs(dst0 + im * istride + r, so[im * n + r]);
            im += q;
            r += rem;
            if (r >= n) {
                r -= n;
                ++im;
            }
        }
        return;
    }
    const int y0 = i0 * m;
    const int orows = min(ntr * m, g.Ho - y0);
    for (int im = 0; im < nimg; ++im) {
        float *dst = out + (((size_t)(b + im) * g.Cout + co) * g.Ho + y0) * g.Wo;
        const float *src = so + (size_t)im * ntr * m * SWo;
        store_strip(dst, src, orows, g.Wo, SWo);
    }
}


template <int T, int FT>
cudaError_t launch_nk2_fft(const Geometry &g, const float *src, float *dst, cudaStream_t s) {
    constexpr int H = FftCfg<T>::H;
    const unsigned nblk = (unsigned)((g.BN + FT - 1) / FT);
    const size_t smem = sizeof(float2) * FT * FftCfg<T>::S2;
    fc_smem_attr((const void *)nk2_fft<T, FT>, (int)smem);
    // channel-fastest grid (measured faster); float2 row loads when tile rows are 8-byte aligned
    const int v2 = (((g.W | g.m) & 1) == 0 && (reinterpret_cast<uintptr_t>(src) & 7) == 0) ? 2 : 0;
    // small tiles (t <= 12) and the 16-tile CTAs of small grids: CTAs of exactly max(row
    // pairs, columns) x 32 threads -- one item each, no idle warps (VGG-3.2 t = 10 NK2 -7%,
    // deep t = 9 -6%; 5x5 t = 18 at 160 instead of 256 threads 66 -> 63.5 us, r02n A/B);
    // larger 32-tile CTAs keep 256 (t = 16 at 288 threads: one CTA fewer per SM, VGG-1.2
    // m = 14 +5%)
    constexpr int RPc = (T + 1) / 2, ITEMS = (RPc > H ? RPc : H) * FT;
    const int nthr = ((T <= 12 || FT < FTN) && ITEMS <= 256) ? (ITEMS + 31) / 32 * 32 : 256;
    if (nblk <= 65535)
        nk2_fft<T, FT><<<dim3(g.C, nblk), nthr, smem, s>>>(g, src, dst, 1 | v2);
    else
        nk2_fft<T, FT><<<dim3(nblk, g.C), nthr, smem, s>>>(g, src, dst, v2);
    return cudaGetLastError();
}

template <int T>
cudaError_t launch_fft(const Geometry &g, const float *src, float *dst, bool forward, cudaStream_t s) {
    constexpr int H = FftCfg<T>::H;
    if (forward) {
        // 16-tile CTAs when 32-tile ones would make fewer than 16 per SM over the whole grid
        // (small layers: wave quantisation; 5x5 t = 18 NK2 64 -> 56 us); otherwise 32 tiles,
        // each (z, channel) row of U a 128-byte run (VGG-1.2 t = 16 NK2 0.42 ms at 16 vs 0.37)
        const long long ctas32 = (long long)g.C * ((g.BN + FTN - 1) / FTN);
        if (ctas32 < 16LL * fc_num_sms()) return launch_nk2_fft<T, 16>(g, src, dst, s);
        return launch_nk2_fft<T, FTN>(g, src, dst, s);
    } else {
        // tiles per CTA ~ 512 / H (one phase-A item per thread), shared memory <= ~100 KB;
        // whole images when they fit (IPC images), else strips of R tile rows
        const int Sm = (g.m * H) % 2 ? g.m * H : g.m * H + 1;
        // staged output pitch: n_w m rounded up to 16 bytes when the output rows are (vector copy-out)
        const int SWo = (g.Wo & 3) == 0 ? (g.n_w * g.m + 3) & ~3 : g.n_w * g.m;
        auto smem_of = [&](int ipc, int r) {
            return (((size_t)ipc * r * g.n_w * Sm + 1) & ~(size_t)1) * sizeof(float2) +
                   (size_t)ipc * r * g.m * SWo * sizeof(float);
        };
        constexpr int items_env = 256;
        // at least 32 tiles per CTA: each (l, c') run of X a warp loads is then >= 128 bytes
        // (VGG-1.2 m = 14 had 16-tile strips: 64-byte runs)
        // (t > 18: at least 16 -- more, smaller CTAs overlap their load and FFT phases; VGG-3.2
        // t = 21 NK4 203 -> 158 us, t = 27 / 32 unchanged, t = 16 VGG-1.2 +3% at 16)
        constexpr int min_tiles = T > 18 ? 16 : 32;
        const int target = items_env / H > min_tiles ? items_env / H : min_tiles;
        int R = target / g.n_w > 0 ? target / g.n_w : 1, IPC = 1;
        if (R >= g.n_h) {
            R = g.n_h;
            IPC = target / g.N > 1 ? target / g.N : 1;
            if (IPC > g.B) IPC = g.B;
        }
        while (IPC > 1 && smem_of(IPC, R) > 100 * 1024) --IPC;
        while (R > 1 && smem_of(IPC, R) > 100 * 1024) --R;
        const size_t smem = smem_of(IPC, R);
        if (smem > 200 * 1024) return cudaErrorInvalidValue;
        fc_smem_attr((const void *)nk4_fft<T>, 200 * 1024);
        const int nstrip = (g.n_h + R - 1) / R;
        const int ngroup = (g.B + IPC - 1) / IPC;
        const int items = H * IPC * R * g.n_w;
        const int threads = items >= 512 ? 512 : (items + 31) / 32 * 32;
        if (ngroup > 65535 || g.Cout > 65535) return cudaErrorInvalidConfiguration;
        nk4_fft<T><<<dim3(nstrip, ngroup, g.Cout), threads, smem, s>>>(g, R, IPC, SWo, src, dst);
    }
    return cudaGetLastError();
}


}  // namespace fcfft
