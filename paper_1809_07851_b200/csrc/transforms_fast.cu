// Fast NK2 / NK4 tile transforms, specialised on the tile edge t at compile time.
//
//  * Winograd (t <= 8): one thread per (channel, tile), the t x t tile in
//    registers, U = B^T d B and Y = A^T X A as unrolled dense products whose
//    matrix entries sit in the kernel-parameter constant bank (Eq. 4).
//  * FFT (Regular and Gauss): a CTA owns 32 consecutive tiles of one channel.
//    Row pass: each thread packs two real tile rows into one complex FFT of
//    length t and splits the half spectra (real-input trick); column pass: one
//    complex FFT of length t per (half-spectrum column, tile) from shared memory
//    (P:1062-1069 half spectrum; P:501-515 arbitrary sizes).  Inverse: pruned
//    column IFFT (keep rows a < m), then two cropped rows per complex IFFT with
//    the self-conjugate bins' imaginary parts dropped (readings R5-R7).
//
// Stores of U and loads of X run along the tile index n (lanes = consecutive
// tiles), so every warp access to the big intermediates is a 128-byte line.
#include <cstdlib>
#include <mutex>

#include "common.h"
#include "fft_tile.cuh"
#include "winograd_tables.h"
#include "xform_util.cuh"

using fct::cf;

using namespace fcx;

namespace {

struct WinoMats {
    float BT[64];
    float AT[64];
};

// ----------------------------------------------------------- Winograd NK1 ---
// One thread per (c', c) kernel (lanes along c: coalesced V stores), V = G g G^T
// fully unrolled for compile-time (t, r); 3xTF32 split written alongside.
struct GMat {
    float G[64];
};

// NC channels per thread: 1 (fp32 / 3xTF32 stores, 128 B per warp store) or 2 (F16X3:
// the pair (c, c+1) written as half2 so a warp store still covers 128 B).
template <int T, int R, int NC>
__global__ void __launch_bounds__(256) nk1_wino(Geometry g, const float *__restrict__ w,
                                                float *__restrict__ V, float *__restrict__ Vlo, int split) {
    constexpr wtab::Tables tg = wtab::make(T - R + 1, R);  // G as literals
    // F16X3 (split 2): CTAs own one output channel c' (its scale first) x a block of channel
    // pairs; otherwise one thread per (c', c)
    int co, c;
    float sv = 1.f;
    if (split == 2) {
        co = blockIdx.x;
        sv = fc_row_vscale(g, w, co);
        c = NC * (blockIdx.y * blockDim.x + threadIdx.x);
        if (c >= g.C) return;
    } else {
        const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
        if (idx >= (long long)g.C * g.Cout) return;
        co = (int)(idx / g.C);
        c = (int)(idx - (long long)co * g.C);
    }
    float tmp[NC][R][T];  // tmp[p][l] = sum_q k[p][q] G[l][q]
#pragma unroll
    for (int j = 0; j < NC; ++j) {
        float k[R][R];
        const bool ok = c + j < g.C;
        const float *ker = w + ((size_t)co * g.C + c + j) * (R * R);
#pragma unroll
        for (int p = 0; p < R; ++p)
#pragma unroll
            for (int q = 0; q < R; ++q) k[p][q] = ok ? __ldg(ker + p * R + q) : 0.f;
#pragma unroll
        for (int p = 0; p < R; ++p)
#pragma unroll
            for (int l = 0; l < T; ++l) {
                float s = -0.f;
#pragma unroll
                for (int q = 0; q < R; ++q) s = wtab::cfma(tg.G[l][q], k[p][q], s);
                tmp[j][p][l] = s;
            }
    }
    const size_t zstride = (size_t)g.M * g.Kp;
    const size_t off = (size_t)co * g.Kp + c;
#pragma unroll
    for (int kk = 0; kk < T; ++kk)
#pragma unroll
        for (int l = 0; l < T; ++l) {
            float s[NC];
#pragma unroll
            for (int j = 0; j < NC; ++j) {
                s[j] = -0.f;
#pragma unroll
                for (int p = 0; p < R; ++p) s[j] = wtab::cfma(tg.G[kk][p], tmp[j][p][l], s[j]);
            }
            const int e = kk * T + l - g.e_lo;  // element shards: [e_lo, e_hi) relative to e_lo
            if (e < 0 || e >= g.e_hi - g.e_lo) continue;
            if (NC == 2)
                fc_store_v2(V, Vlo, off + (size_t)e * zstride, s[0], s[NC - 1], sv);
            else
                fc_store_v(V, Vlo, off + (size_t)e * zstride, s[0], split, sv);
        }
}
template <int T, int R>
cudaError_t launch_nk1_wino(const Geometry &g, const ConvConsts &hc, const float *w, float *V, float *Vlo,
                            int split, cudaStream_t s) {
    (void)hc;
    const long long n = (long long)g.C * g.Cout;
    if (split == 2) {  // channel pairs (Kp is a multiple of 8: the pad column absorbs an odd C)
        const int np = (g.C + 1) / 2;
        const int bs = np >= 256 ? 256 : (np + 31) / 32 * 32;
        nk1_wino<T, R, 2><<<dim3((unsigned)g.Cout, (unsigned)((np + bs - 1) / bs)), bs, 0, s>>>(g, w, V, Vlo, split);
    } else {
        nk1_wino<T, R, 1><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(g, w, V, Vlo, split);
    }
    return cudaGetLastError();
}

// ----------------------------------------------------------- Winograd NK2 ---
// One thread per (channel, tile): the t x t input tile straight from global
// memory into registers (adjacent lanes = adjacent tiles, so the overlapping
// reads hit L1), U = B^T d B unrolled, t^2 streaming stores along n.  (A
// shared-memory strip-staged variant measured 2.4x slower on VGG-3.2: with the
// load and compute phases separated by a CTA barrier too few loads stay in flight.)
// RED: also reduce max|U| into *g.umax (F16X3 contraction scale); 128-thread CTAs
// capped at 64 registers so the reduction costs no occupancy.
template <int T, bool RED>
// flags bit 0 (cfast): grid (C, n-blocks) -- consecutive CTAs write consecutive channels of
// one U block, i.e. one sequential run of Z * 512 bytes each (U is blocked by FC_TB =
// blockDim tiles); bit 1 (v2): even W and m, 8-byte aligned input -- every tile row starts
// 8-byte aligned, load it as float2 (half the L1 requests of the overlapping lane accesses)
__global__ void __launch_bounds__(RED ? 128 : 512, (RED && T <= 6) ? 8 : (RED ? 4 : 1))
    nk2_wino(Geometry g, const float *__restrict__ in, float *__restrict__ U, int flags) {
    const int cfast = flags & 1;
    constexpr wtab::Tables tb = wtab::make(2, T - 1);  // B^T as literals (depends on t only)
    const long long n_ = (long long)(cfast ? blockIdx.y : blockIdx.x) * blockDim.x + threadIdx.x;
    const int c = cfast ? blockIdx.x : blockIdx.y;
    if (!RED && n_ >= g.BN) return;
    // idle lanes (RED: they take part in the CTA reduction) recompute the last tile and store
    // the same values to the same addresses as its own lane -- no per-store predicate
    const long long n = n_ < g.BN ? n_ : g.BN - 1;
    // BN < 2^31 (U indices): fast divisions by the plan's constants N and n_w
    const int b = fc_div((int)n, g.divN), tile = (int)n - b * g.N;
    const int ti = fc_div(tile, g.divNw), tj = tile - ti * g.n_w;
    const int y0 = ti * g.m, x0 = tj * g.m;
    const float *src = in + ((size_t)b * g.C + c) * g.H * g.W + (size_t)y0 * g.W + x0;
    float d[T][T];
    // (t = 4 keeps scalar loads: float2 measured slower on VGG-1.2 F(2,3), NK2 0.82 -> 0.95+ ms)
    if (T % 2 == 0 && T >= 6 && (flags & 2) && y0 + T <= g.H && x0 + T <= g.W) {
#pragma unroll
        for (int a = 0; a < T; ++a)
#pragma unroll
            for (int q = 0; q < T; q += 2) {
                const float2 v = __ldg(reinterpret_cast<const float2 *>(src + a * g.W + q));
                d[a][q] = v.x;
                d[a][q + 1 < T ? q + 1 : q] = v.y;
            }
    } else if (y0 + T <= g.H && x0 + T <= g.W) {
#pragma unroll
        for (int a = 0; a < T; ++a)
#pragma unroll
            for (int q = 0; q < T; ++q) d[a][q] = __ldg(src + a * g.W + q);
    } else {
#pragma unroll
        for (int a = 0; a < T; ++a)
#pragma unroll
            for (int q = 0; q < T; ++q)
                d[a][q] = (y0 + a < g.H && x0 + q < g.W) ? __ldg(src + a * g.W + q) : 0.f;
    }
    float z[T][T];  // z[a][l] = sum_q d[a][q] BT[l][q]
#pragma unroll
    for (int a = 0; a < T; ++a)
#pragma unroll
        for (int l = 0; l < T; ++l) {
            float s = -0.f;
#pragma unroll
            for (int q = 0; q < T; ++q) s = wtab::cfma(tb.BT[l][q], d[a][q], s);
            z[a][l] = s;
        }
    float *dp = U + fc_u_off(g, n, c, 0);  // element e at dp[e * zs], stepped e by e
    const size_t zs = fc_u_zs(g);
    float umx = 0.f;
#pragma unroll
    for (int k = 0; k < T; ++k)
#pragma unroll
        for (int l = 0; l < T; ++l) {
            float s = -0.f;
#pragma unroll
            for (int a = 0; a < T; ++a) s = wtab::cfma(tb.BT[k][a], z[a][l], s);
            *dp = s;
            dp += zs;
            if (RED) umx = fmaxf(umx, fabsf(s));
        }
    if (RED) {  // per-image max|U| (b0: the image of the CTA's first tile)
        const long long nf = (long long)(cfast ? blockIdx.y : blockIdx.x) * blockDim.x;
        fc_block_umax_img(g.umax, fc_div((int)(nf < g.BN ? nf : g.BN - 1), g.divN), b, umx);
    }
}


// r[q] = sum_l A^T[q][l] x[l] for the compile-time A^T of F(MM, T-MM+1).  The finite
// points are ordered 0, 1, -1, 2, -2, 1/2, -1/2 (wtab::point), so columns (2j+1, 2j+2)
// hold +-p and A^T[q][2j+2] = (-1)^q A^T[q][2j+1]: each pair costs one sum and one
// difference shared by all rows (checked at compile time by at_pairs_ok).
template <int T, int MM>
__host__ __device__ constexpr bool at_pairs_ok() {
    constexpr wtab::Tables ta = wtab::make(MM, T - MM + 1);
    for (int q = 0; q < MM; ++q)
        for (int j = 0; 2 * j + 2 <= T - 2; ++j)
            if (ta.AT[q][2 * j + 2] != ((q & 1) ? -ta.AT[q][2 * j + 1] : ta.AT[q][2 * j + 1])) return false;
    return true;
}

template <int T, int MM>
__device__ __forceinline__ void at_rows(const float *x, float *r) {
    constexpr wtab::Tables ta = wtab::make(MM, T - MM + 1);
    static_assert(at_pairs_ok<T, MM>(), "A^T columns are not +-p pairs");
    constexpr int NP = (T - 2) / 2;
    float sp[NP > 0 ? NP : 1], dp[NP > 0 ? NP : 1];
#pragma unroll
    for (int j = 0; j < NP; ++j) {
        sp[j] = x[2 * j + 1] + x[2 * j + 2];
        dp[j] = x[2 * j + 1] - x[2 * j + 2];
    }
#pragma unroll
    for (int q = 0; q < MM; ++q) {
        float acc = wtab::cfma(ta.AT[q][0], x[0], -0.f);
#pragma unroll
        for (int j = 0; j < NP; ++j) acc = wtab::cfma(ta.AT[q][2 * j + 1], (q & 1) ? dp[j] : sp[j], acc);
        if ((T - 2) & 1) acc = wtab::cfma(ta.AT[q][T - 2], x[T - 2], acc);
        r[q] = wtab::cfma(ta.AT[q][T - 1], x[T - 1], acc);
    }
}

// Y = A^T X A for one tile, X streamed by rows through load_row(k, x[T]) in the order
// 0, (1,2), (3,4), ..., [T-2], T-1: a +-p row pair enters Y as its sum (even output
// rows a) or difference (odd a), as the columns do in at_rows.  Shared by both NK4
// kernels so their results are bit-identical.
template <int T, int MM, typename LoadRow>
__device__ __forceinline__ void wino_out_tile(LoadRow load_row, float (&y)[MM][MM]) {
    constexpr wtab::Tables ta = wtab::make(MM, T - MM + 1);
#pragma unroll
    for (int a = 0; a < MM; ++a)
#pragma unroll
        for (int q = 0; q < MM; ++q) y[a][q] = -0.f;
    auto add_row = [&](int k, const float *r) {
#pragma unroll
        for (int a = 0; a < MM; ++a)
#pragma unroll
            for (int q = 0; q < MM; ++q) y[a][q] = wtab::cfma(ta.AT[a][k], r[q], y[a][q]);
    };
    {
        float x[T], r[MM];
        load_row(0, x);
        at_rows<T, MM>(x, r);
        add_row(0, r);
    }
#pragma unroll
    for (int j = 0; 2 * j + 2 <= T - 2; ++j) {
        float x1[T], x2[T], r1[MM], r2[MM], rs[MM], rd[MM];
        load_row(2 * j + 1, x1);
        load_row(2 * j + 2, x2);
        at_rows<T, MM>(x1, r1);
        at_rows<T, MM>(x2, r2);
#pragma unroll
        for (int q = 0; q < MM; ++q) {
            rs[q] = r1[q] + r2[q];
            rd[q] = r1[q] - r2[q];
        }
#pragma unroll
        for (int a = 0; a < MM; ++a)
#pragma unroll
            for (int q = 0; q < MM; ++q) y[a][q] = wtab::cfma(ta.AT[a][2 * j + 1], (a & 1) ? rd[q] : rs[q], y[a][q]);
        asm volatile("" ::: "memory");  // keep about one row pair of loads in flight
    }
    if ((T - 2) & 1) {
        float x[T], r[MM];
        load_row(T - 2, x);
        at_rows<T, MM>(x, r);
        add_row(T - 2, r);
    }
    {
        float x[T], r[MM];
        load_row(T - 1, x);
        at_rows<T, MM>(x, r);
        add_row(T - 1, r);
    }
}

// ----------------------------------------------------------- Winograd NK4 ---
// CTA = (strip of R tile rows, image group, output channel c').  One thread per tile
// loads its t^2 elements of X along n, computes Y = A^T X A, and writes the m x m
// block into a shared-memory output strip; the CTA then stores the strip's
// contiguous output rows with coalesced writes (crop to Ho x Wo on the way).
template <int T, int MM>
__global__ void __launch_bounds__(256, 4) nk4_wino(Geometry g, int R, int IPC, int SWo,
                                                const float *__restrict__ X, float *__restrict__ out) {
    constexpr wtab::Tables ta = wtab::make(MM, T - MM + 1);  // A^T as literals
    extern __shared__ float so[];  // [img][ntr*m][SWo]
    const int m = g.m;
    // blockIdx.x = (image group, strip); IPC > 1 only with whole-image strips (R = n_h)
    const int strip = blockIdx.x, b = blockIdx.y * IPC, co = blockIdx.z;  // grid (strips, image groups, C')
    const int i0 = strip * R;
    const int ntr = min(R, g.n_h - i0);
    const int nimg = min(IPC, g.B - b);
    const int ntiles = nimg * ntr * g.n_w;  // contiguous in n
    const long long nbase = ((long long)b * g.n_h + i0) * g.n_w;
    // whole images of narrow rows per CTA (R = n_h, Wo < 48): stage the cropped planes at
    // pitch Wo and copy each image out as one flat run -- the per-image strip copies were ~70%
    // of the deep layer's NK4 instructions (ncu r02 deep: NK4 34 -> 18 us).  Wide rows keep
    // the padded-pitch vector staging (VGG-3.2 F(6,3) NK4 131 -> 156 us with the cropped one).
    const bool whole = R == g.n_h && g.Wo < 48;
    const float inv_nh = 1.f / (float)g.n_h;
    size_t ebytes = (size_t)g.Xm * g.BN_pad * sizeof(float);
    asm("" : "+l"(ebytes));
    const float *src0 = X + (size_t)co * g.BN_pad + nbase;
    for (int tl = threadIdx.x; tl < ntiles; tl += blockDim.x) {
        // stream the tile by rows of X (one row pair live at a time: registers / occupancy)
        float y[MM][MM];
        // element e = k T + l at sp[e * estride]; wino_out_tile asks for the rows in
        // increasing k, so step the pointer by an opaque byte stride (one 64-bit add per
        // load instead of a re-derived 64-bit index product)
        const char *sp = reinterpret_cast<const char *>(src0 + tl);
        wino_out_tile<T, MM>(
            [&](int k, float *x) {
                (void)k;
#pragma unroll
                for (int l = 0; l < T; ++l) {
                    x[l] = __ldcs(reinterpret_cast<const float *>(sp));
                    sp += ebytes;
                }
            },
            y);
        const int ti = fc_div(tl, g.divNw), tj = tl - ti * g.n_w;  // ti counts rows across the CTA's images
        if (whole) {  // whole images: stage the cropped Ho x Wo planes back to back
            const int im = fcx::fc_sdiv(ti, inv_nh), oy = (ti - im * g.n_h) * m, ox = tj * m;
            float *q = so + ((size_t)im * g.Ho + oy) * g.Wo + ox;
#pragma unroll
            for (int a = 0; a < MM; ++a)
#pragma unroll
                for (int c = 0; c < MM; ++c)
                    if (oy + a < g.Ho && ox + c < g.Wo) q[a * g.Wo + c] = y[a][c];
            continue;
        }
        float *q0 = so + ti * m * SWo + tj * m;
#pragma unroll
        for (int a = 0; a < MM; ++a) {
            if (MM % 4 == 0 && (SWo & 3) == 0) {  // 16-byte rows: conflict-free vector stores
#pragma unroll
                for (int q = 0; q < MM; q += 4)
                    *reinterpret_cast<float4 *>(q0 + a * SWo + q) =
                        make_float4(y[a][q], y[a][(q + 1) % MM], y[a][(q + 2) % MM], y[a][(q + 3) % MM]);
            } else if (MM % 2 == 0 && (SWo & 1) == 0) {
#pragma unroll
                for (int q = 0; q < MM; q += 2)
                    *reinterpret_cast<float2 *>(q0 + a * SWo + q) = make_float2(y[a][q], y[a][(q + 1) % MM]);
            } else {
#pragma unroll
                for (int q = 0; q < MM; ++q) q0[a * SWo + q] = y[a][q];
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

// F16X3 scale prologue for the z-sliced FFT NK1: one CTA per output channel c'
// (fc_row_vscale: max|W[c']| -> s_v[c'], 1/s_v[c']).
__global__ void __launch_bounds__(256) nk1_row_scale(Geometry g, const float *__restrict__ w) {
    fc_row_vscale(g, w, blockIdx.x);
}

// ---------------------------------------------------------------- FFT NK1 ---
// One thread per (c', c) kernel, V = conj(DFT2(pad_t(g))) / t^2 with the
// zero-padded r x r kernel (only r rows / columns contribute),
// unrolled for compile-time (t, r) with constant-memory twiddles; the real
// embedding (Regular) or the Gauss pre-sums and the 3xTF32 split are written
// along c (coalesced).
template <int T, int R, int NC>
__global__ void __launch_bounds__(128) nk1_fft(Geometry g, const float *__restrict__ w, float *__restrict__ V,
                                               float *__restrict__ Vlo, int split) {
    constexpr int H = T / 2 + 1;
    // one thread per (c', NC channels) and one half-spectrum column l per grid z-slice;
    // F16X3's per-c' scale comes from nk1_row_scale (launched first), not from an
    // in-CTA reduction that every z-slice would repeat.  NC = 2: half2 pair stores.
    const int npc = (g.C + NC - 1) / NC;
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (long long)npc * g.Cout) return;
    const int co = (int)(idx / npc), c = NC * (int)(idx - (long long)co * npc);
    const float sv = split == 2 ? g.vscale[co] : 1.f;
    const int l = blockIdx.z;
    const float inv = 1.0f / ((float)T * (float)T);
    cf tr[NC][R];  // row DFT along q: sum_q g[p][q] W^{-l q}
#pragma unroll
    for (int j = 0; j < NC; ++j) {
        float k[R][R];
        const bool ok = c + j < g.C;
        const float *ker = w + ((size_t)co * g.C + c + j) * (R * R);
#pragma unroll
        for (int p = 0; p < R; ++p)
#pragma unroll
            for (int q = 0; q < R; ++q) k[p][q] = ok ? __ldg(ker + p * R + q) : 0.f;
#pragma unroll
        for (int p = 0; p < R; ++p) {
            float ar = k[p][0], ai = 0.f;
#pragma unroll
            for (int q = 1; q < R; ++q) {
                const int jj = (l * q) % T;
                const float2 tw = fct::c_tw[fct::tw_base(T) + jj];
                ar = fmaf(k[p][q], tw.x, ar);
                ai = fmaf(-k[p][q], tw.y, ai);
            }
            tr[j][p] = cf{ar, ai};
        }
    }
    const size_t zstride = (size_t)(g.cplx ? g.Cout : g.M) * g.Kp;
    auto put = [&](size_t o, const float *v) {
        if (NC == 2)
            fc_store_v2(V, Vlo, o, v[0], v[NC - 1], sv);
        else
            fc_store_v(V, Vlo, o, v[0], split, sv);
    };
    // offsets: ez = e * zstride for e = kk * H + l, stepped by an opaque H * zstride (one
    // 64-bit add per kk instead of 64-bit index products per store)
    size_t hz = (size_t)H * zstride;
    asm("" : "+l"(hz));
    // element shards write e in [e_lo, e_hi) relative to e_lo (the whole E otherwise)
    const int elo = g.e_lo, ecnt = g.e_hi - g.e_lo;
    size_t ez = (size_t)(l - elo) * zstride;
    const size_t o00 = (size_t)co * g.Kp + c;                          // (c', c)
    const size_t o01 = o00 + g.C, o10 = o00 + (size_t)g.Cout * g.Kp;  // (c', C + c), (C' + c', c)
    const size_t o11 = o10 + g.C, gpl = (size_t)ecnt * zstride;
#pragma unroll
    for (int kk = 0; kk < T; ++kk, ez += hz) {
        if ((unsigned)(kk * H + l - elo) >= (unsigned)ecnt) continue;
        float vr[NC], vi[NC], t0[NC], t1[NC];
#pragma unroll
        for (int j = 0; j < NC; ++j) {
            cf acc = tr[j][0];
#pragma unroll
            for (int p = 1; p < R; ++p) {
                const cf t = fct::twiddle_mul<T, -1>(tr[j][p], kk * p);
                acc.x += t.x;
                acc.y += t.y;
            }
            vr[j] = acc.x * inv;  // conj(DFT) / t^2
            vi[j] = -acc.y * inv;
        }
        if (g.method == CONV_REGULAR_FFT && g.cplx) {  // (V_r, V_i) planes z = 2e, 2e + 1
            put(2 * ez + o00, vr);
            put(2 * ez + zstride + o00, vi);
        } else if (g.method == CONV_REGULAR_FFT) {  // real embedding [[V_r, -V_i], [V_i, V_r]]
#pragma unroll
            for (int j = 0; j < NC; ++j) t0[j] = -vi[j];
            put(ez + o00, vr);
            put(ez + o01, t0);
            put(ez + o10, vi);
            put(ez + o11, vr);
        } else {  // Gauss: V_r, V_i - V_r, V_r + V_i in planes z = e, E + e, 2E + e
#pragma unroll
            for (int j = 0; j < NC; ++j) {
                t0[j] = vi[j] - vr[j];
                t1[j] = vr[j] + vi[j];
            }
            put(ez + o00, vr);
            put(ez + gpl + o00, t0);
            put(ez + 2 * gpl + o00, t1);
        }
    }
}

template <int T, int R>
cudaError_t launch_nk1_fft(const Geometry &g, const float *w, float *V, float *Vlo, int split, cudaStream_t s) {
    const long long n = (long long)g.C * g.Cout;
    constexpr int H = T / 2 + 1;
    if (split == 2) {
        nk1_row_scale<<<(unsigned)g.Cout, 256, 0, s>>>(g, w);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    // F16X3 with even C: channel pairs (the real embedding's second column block starts at C)
    if (split == 2 && g.C % 2 == 0) {
        const long long np = (long long)(g.C / 2) * g.Cout;
        nk1_fft<T, R, 2><<<dim3((unsigned)((np + 127) / 128), 1, H), 128, 0, s>>>(g, w, V, Vlo, split);
    } else {
        nk1_fft<T, R, 1><<<dim3((unsigned)((n + 127) / 128), 1, H), 128, 0, s>>>(g, w, V, Vlo, split);
    }
    return cudaGetLastError();
}

// tile rows per CTA: the staged strip stays within ~32 KB of shared memory
inline int wino_strip_rows(const Geometry &g, int row_floats) {
    const int per_tile_row = g.m * row_floats * 4;
    int R = (32 * 1024 - (g.r - 1) * row_floats * 4) / per_tile_row;
    R = R < 1 ? 1 : R;
    const int max_tiles = 1024;
    if (R * g.n_w > max_tiles) R = max_tiles / g.n_w > 0 ? max_tiles / g.n_w : 1;
    return R < g.n_h ? R : g.n_h;
}

template <int T, int MM>
cudaError_t launch_wino(const Geometry &g, const float *src, float *dst, bool forward, cudaStream_t s) {
    if (forward) {
        {
            // 128-tile CTAs (one U block), channel-fastest grid (measured faster than n-fastest)
            constexpr int bs = FC_TB;
            const int v2 = (((g.W | g.m) & 1) == 0 && (reinterpret_cast<uintptr_t>(src) & 7) == 0) ? 2 : 0;
            if (g.umax) {
                const unsigned nblk = (unsigned)((g.BN + 127) / 128);
                if (nblk <= 65535)
                    nk2_wino<T, true><<<dim3(g.C, nblk), 128, 0, s>>>(g, src, dst, 1 | v2);
                else
                    nk2_wino<T, true><<<dim3(nblk, g.C), 128, 0, s>>>(g, src, dst, v2);
            } else {
                const unsigned nblk = (unsigned)((g.BN + bs - 1) / bs);
                if (nblk <= 65535)
                    nk2_wino<T, false><<<dim3(g.C, nblk), bs, 0, s>>>(g, src, dst, 1 | v2);
                else
                    nk2_wino<T, false><<<dim3(nblk, g.C), bs, 0, s>>>(g, src, dst, v2);
            }
        }
    } else {
        // about 256 tiles per CTA: strips of one image, or several whole images
        const int SWo = (g.Wo & 3) == 0 ? (g.n_w * g.m + 3) & ~3 : g.n_w * g.m;  // 16-byte staged rows
        constexpr int target = 256;
        int R = wino_strip_rows(g, SWo), IPC = 1;
        if (R * g.n_w > target) R = target / g.n_w > 0 ? target / g.n_w : 1;
        if (R >= g.n_h) {
            R = g.n_h;
            IPC = target / g.N > 1 ? target / g.N : 1;
            if (IPC > g.B) IPC = g.B;
            while (IPC > 1 && (size_t)IPC * R * g.m * SWo * sizeof(float) > 100 * 1024) --IPC;
        }
        const int nstrip = (g.n_h + R - 1) / R;
        const int ngroup = (g.B + IPC - 1) / IPC;
        // whole images (R = n_h): the kernel stages cropped Ho x Wo planes, at most the strip size
        const size_t smem = sizeof(float) * (size_t)IPC * R * g.m * SWo;
        if (smem > 200 * 1024) return cudaErrorInvalidValue;
        fc_smem_attr((const void *)nk4_wino<T, MM>, 200 * 1024);
        const int tiles = IPC * R * g.n_w;
        const int threads = tiles >= 256 ? 256 : (tiles + 31) / 32 * 32;
        if (ngroup > 65535 || g.Cout > 65535) return cudaErrorInvalidConfiguration;
        nk4_wino<T, MM><<<dim3(nstrip, ngroup, g.Cout), threads, smem, s>>>(g, R, IPC, SWo, src, dst);
    }
    return cudaGetLastError();
}

cudaError_t dispatch(const Geometry &g, const ConvConsts &hc, const float *src, float *dst, bool forward,
                     cudaStream_t s, bool *handled) {
    *handled = true;
    if (g.method == CONV_WINOGRAD) {
        (void)hc;
        // (t, m) pairs with compile-time matrices; others use the runtime-matrix kernels
#define FC_WINO_CASE(TT, MM) \
    if (g.t == TT && g.m == MM) return launch_wino<TT, MM>(g, src, dst, forward, s);
        FC_WINO_TILES(FC_WINO_CASE)
#undef FC_WINO_CASE
        *handled = false;
        return cudaSuccess;
    }
    // FFT NK2 / NK4 codelets live in three translation units by tile size (parallel builds)
    int h = 0;
    cudaError_t e = fc_fft_xform_a(g, src, dst, forward, s, &h);
    if (!h) e = fc_fft_xform_b(g, src, dst, forward, s, &h);
    if (!h) e = fc_fft_xform_c(g, src, dst, forward, s, &h);
    *handled = h != 0;
    return h ? e : cudaSuccess;
}

}  // namespace

cudaError_t fc_init_twiddles() {
    cudaError_t e = fct::upload_twiddles();  // NK1 FFT (this unit)
    if (e == cudaSuccess) e = fc_fft_twiddles_a();
    if (e == cudaSuccess) e = fc_fft_twiddles_b();
    if (e == cudaSuccess) e = fc_fft_twiddles_c();
    return e;
}

cudaError_t fc_launch_kernel_transform_fast(const Geometry &g, const ConvConsts &hc, const float *w, float *V,
                                            float *Vlo, int split, cudaStream_t s, int *handled) {
    *handled = 1;
    if (g.method == CONV_WINOGRAD) {
#define FC_NK1W_CASE(TT, MM) \
    if (g.t == TT && g.m == MM) return launch_nk1_wino<TT, TT - MM + 1>(g, hc, w, V, Vlo, split, s);
        FC_WINO_TILES(FC_NK1W_CASE)
#undef FC_NK1W_CASE
    } else if (g.r == 3) {  // every FFT tile edge with NK2 / NK4 codelets (FC_FFT_TILES)
        switch (g.t) {
#define FC_NK1_CASE(TT) \
    case TT: return launch_nk1_fft<TT, 3>(g, w, V, Vlo, split, s);
            FC_FFT_TILES(FC_NK1_CASE)
#undef FC_NK1_CASE
        }
    } else if (g.r == 5) {
        switch (g.t) {
#define FC_NK1_CASE(TT) \
    case TT: if (TT >= 5) return launch_nk1_fft<(TT >= 5 ? TT : 5), 5>(g, w, V, Vlo, split, s); break;
            FC_FFT_TILES(FC_NK1_CASE)
#undef FC_NK1_CASE
        }
    }
    *handled = 0;
    return cudaSuccess;
}

cudaError_t fc_launch_transform_fast(const Geometry &g, const ConvConsts &hc, const float *src, float *dst,
                                     int forward, cudaStream_t s, int *handled) {
    bool h = false;
    cudaError_t e = dispatch(g, hc, src, dst, forward != 0, s, &h);
    *handled = h ? 1 : 0;
    return e;
}

int fc_fast_transforms(int method, int t, int m, int r) {
    if (method == CONV_WINOGRAD) {
#define FC_WINO_HAVE(TT, MM) \
    if (t == TT && m == MM) return 1;
        FC_WINO_TILES(FC_WINO_HAVE)
#undef FC_WINO_HAVE
        return 0;
    }
    if (method != CONV_REGULAR_FFT && method != CONV_GAUSS_FFT) return 0;
    (void)m;
    (void)r;
    switch (t) {
#define FC_FFT_HAVE(TT) \
    case TT: return 1;
        FC_FFT_TILES(FC_FFT_HAVE)
#undef FC_FFT_HAVE
    }
    return 0;
}

// kernel launches of NK1 for this geometry: the FFT codelets with the F16X3 split run a
// per-c' scale prologue first (2), everything else one kernel
int fc_nk1_launches(const Geometry &g, int split) {
    if (g.nd || g.method == CONV_WINOGRAD || g.method == CONV_DIRECT || split != 2) return 1;
    if (g.r != 3 && g.r != 5) return 1;
    if (g.r == 5 && g.t < 5) return 1;
    return fc_fast_transforms(g.method, g.t, g.m, g.r) ? 2 : 1;
}
