// C-ABI of the fastconv library (include/fastconv.h): plan geometry, exact
// Winograd matrices, DFT twiddles, workspace layout, and stage dispatch.
//
// Geometry follows PAPER.md P:956-965 (t = m + r - 1, N = ceil((x-r+1)/m)^2
// per image, generalised to H != W), the half-spectrum width P:1062-1065
// (t * ceil((t+1)/2) stored complex numbers = t * (t/2 + 1)), and the stage
// costs of Table "layer-stuff" P:1008-1042.
#include <math.h>

#include <cmath>
#include <vector>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <new>

#include <mutex>
#include <algorithm>
#include <map>
#include <set>

#include "common.h"

static thread_local char g_err[512] = "";

void fc_set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

// ---------------------------------------------------------------------------
// Exact rational Winograd matrices (PAPER.md P:274-290
// "derived from Vandermonde matrices for Homogeneous Coordinate polynomials").
// Points {0, 1, -1, 2, -2, 1/2, -1/2, ...} truncated to t-1 finite points plus
// the point at infinity (reading R8).  With V the t x t evaluation
// matrix of degree-<t polynomials (infinity row = leading coefficient), and
// V_r, V_m its degree-<r / degree-<m analogues, correlation is the transpose
// of polynomial multiplication:  y = V_m^T [ (V_r g) . (V^-T d) ], i.e.
// A^T = V_m^T, G = V_r, B^T = V^-T; row i of B^T is scaled by the lcm of its
// denominators and row i of G divided by it.
// ---------------------------------------------------------------------------
namespace {
struct Frac {
    long long n, d;
};
long long gcdll(long long a, long long b) {
    if (a < 0) a = -a;
    if (b < 0) b = -b;
    while (b) {
        long long t = a % b;
        a = b;
        b = t;
    }
    return a ? a : 1;
}
Frac mk(long long n, long long d) {
    if (d < 0) { n = -n; d = -d; }
    long long g = gcdll(n, d);
    return Frac{n / g, d / g};
}
Frac sub(Frac a, Frac b) { return mk(a.n * b.d - b.n * a.d, a.d * b.d); }
Frac mul(Frac a, Frac b) { return mk(a.n * b.n, a.d * b.d); }
Frac dvd(Frac a, Frac b) { return mk(a.n * b.d, a.d * b.n); }
double val(Frac a) { return (double)a.n / (double)a.d; }
}  // namespace

conv_status fc_winograd_rational(int m, int r, double *AT, double *BT, double *G) {
    const int t = m + r - 1;
    if (m < 2 || r < 2 || t > 8) {
        fc_set_error("Winograd F(%d,%d): need m>=2, r>=2, t=m+r-1<=8", m, r);
        return CONV_ERR_UNSUPPORTED;
    }
    static const Frac pts[7] = {{0, 1}, {1, 1}, {-1, 1}, {2, 1}, {-2, 1}, {1, 2}, {-1, 2}};
    Frac V[8][8], Inv[8][8];
    for (int i = 0; i < t; ++i)
        for (int j = 0; j < t; ++j) {
            if (i < t - 1) {
                Frac p = {1, 1};
                for (int e = 0; e < j; ++e) p = mul(p, pts[i]);
                V[i][j] = p;
            } else {
                V[i][j] = mk(j == t - 1 ? 1 : 0, 1);  // infinity: leading coefficient
            }
            Inv[i][j] = mk(i == j ? 1 : 0, 1);
        }
    // Gauss-Jordan inverse in exact rationals
    for (int col = 0; col < t; ++col) {
        int piv = col;
        while (piv < t && V[piv][col].n == 0) ++piv;
        if (piv == t) {
            fc_set_error("singular Vandermonde matrix");
            return CONV_ERR_UNSUPPORTED;
        }
        for (int j = 0; j < t; ++j) {
            Frac x = V[col][j]; V[col][j] = V[piv][j]; V[piv][j] = x;
            x = Inv[col][j]; Inv[col][j] = Inv[piv][j]; Inv[piv][j] = x;
        }
        Frac d = V[col][col];
        for (int j = 0; j < t; ++j) {
            V[col][j] = dvd(V[col][j], d);
            Inv[col][j] = dvd(Inv[col][j], d);
        }
        for (int i = 0; i < t; ++i) {
            if (i == col || V[i][col].n == 0) continue;
            Frac f = V[i][col];
            for (int j = 0; j < t; ++j) {
                V[i][j] = sub(V[i][j], mul(f, V[col][j]));
                Inv[i][j] = sub(Inv[i][j], mul(f, Inv[col][j]));
            }
        }
    }
    // B^T = (V^-1)^T : BT[i][j] = Inv[j][i]
    Frac bt[8][8], gm[8][8];
    for (int i = 0; i < t; ++i)
        for (int j = 0; j < t; ++j) bt[i][j] = Inv[j][i];
    // G = V_r (t x r), infinity row selects coefficient r-1
    for (int i = 0; i < t; ++i)
        for (int j = 0; j < r; ++j) {
            if (i < t - 1) {
                Frac p = {1, 1};
                for (int e = 0; e < j; ++e) p = mul(p, pts[i]);
                gm[i][j] = p;
            } else {
                gm[i][j] = mk(j == r - 1 ? 1 : 0, 1);
            }
        }
    // row scaling: move denominators of B^T rows into G rows
    for (int i = 0; i < t; ++i) {
        long long L = 1;
        for (int j = 0; j < t; ++j) L = L / gcdll(L, bt[i][j].d) * bt[i][j].d;
        for (int j = 0; j < t; ++j) bt[i][j] = mul(bt[i][j], mk(L, 1));
        for (int j = 0; j < r; ++j) gm[i][j] = dvd(gm[i][j], mk(L, 1));
    }
    // A^T = V_m^T (m x t)
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < t; ++j) {
            Frac p;
            if (j < t - 1) {
                p = Frac{1, 1};
                for (int e = 0; e < i; ++e) p = mul(p, pts[j]);
            } else {
                p = mk(i == m - 1 ? 1 : 0, 1);
            }
            AT[i * t + j] = val(p);
        }
    for (int i = 0; i < t; ++i) {
        for (int j = 0; j < t; ++j) BT[i * t + j] = val(bt[i][j]);
        for (int j = 0; j < r; ++j) G[i * r + j] = val(gm[i][j]);
    }
    return CONV_OK;
}

// ---------------------------------------------------------------------------
// Geometry + algorithmic cost
// ---------------------------------------------------------------------------
static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

cudaError_t fc_smem_attr(const void *func, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({func, dev})) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.insert({func, dev});
    return e;
}

int fc_max_clusters(const void *func, const cudaLaunchConfig_t *cfg) {
    static std::mutex mu;
    static std::map<std::pair<const void *, int>, int> cache;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({func, dev});
    if (it != cache.end()) return it->second;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, func, cfg) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    cache[{func, dev}] = n;
    return n;
}

int fc_num_sms() {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return 148;
    return n;
}

Geometry fc_chunk_geometry(const Geometry &g, int Bc) {
    Geometry c = g;
    c.B = Bc;
    c.BN = (long long)Bc * g.N;
    c.BN_pad = (c.BN + FC_TB - 1) / FC_TB * FC_TB;
    return c;
}

// Gauss epilogue combine: it saves one of X's three planes in NK3's writes and
// NK4's reads, but three accumulators fit TMEM only as 128-column tiles, and those run the
// F16X3 contraction ~1.35x slower per FLOP than 256-column tiles (per-SM operand traffic:
// V' is re-staged per 128 columns).  Decide by the paper's stage-sum model for
// NK3 + NK4 with B200 constants measured on this kernel set (profiles/r01_summary.md);
// conv_plan_options.gauss_combine forces the choice.  G: Z, K, E, BN filled, Gauss-FFT.
static bool gauss_combine_pays(const Geometry &G, int force) {
    if (force >= 0) return force != 0;
    const double bw = 6.5e12, bw4 = 4.9e12;     // HBM: streaming / NK4's achieved
    const double r256 = 1.3e15, r128 = 0.95e15;  // F16X3 issue rate (3 fp16 products / FLOP)
    const double BN = (double)G.BN, E = G.E, C = G.C, Co = G.Cout;
    const double pad256 = std::ceil(BN / 256.0) * 256.0, pad128 = std::ceil(BN / 128.0) * 128.0;
    const double mma = 3.0 * 6.0 * E * C * Co;  // tensor FLOPs per padded column
    const double u = 4.0 * 3.0 * E * BN * C, x3 = 4.0 * 3.0 * E * BN * Co, x2 = x3 * 2.0 / 3.0;
    const double o = 4.0 * G.B * Co * (double)G.vout;
    // the 3-plane contraction also drops to 128-column tiles when 256 would pad B N by >= 25%
    const double r3 = 4.0 * pad256 >= 5.0 * pad128 ? mma * pad128 / r128 : mma * pad256 / r256;
    const double t3 = std::max(r3, (u + x3) / bw) + (x3 + o) / bw4;
    const double tgc = std::max(mma * pad128 / r128, (u + x2) / bw) + (x2 + o) / bw4;
    return tgc < t3;
}

// Optional batch chunking (conv_plan_options.chunk_images): NK2 -> NK3 -> NK4 per group of
// images so that a chunk's U and X could stay in the 126 MB L2.  Off by default: on VGG-3.2
// (F(4,3)) chunks of 2/4/6/8 images measured 2.5x / 1.7x / 1.5x / 1.4x slower than one pass
// (smaller launches pay wave tails and partial contraction tiles; profiles/r01_summary.md).
static int pick_chunk(const Geometry &G, int chunk_images) {
    if (G.method == CONV_DIRECT || chunk_images <= 0 || chunk_images > G.B) return G.B;
    return chunk_images;
}

static conv_status check_options(const conv_plan_options *o) {
    if (o->struct_size != (int)sizeof(conv_plan_options)) {
        fc_set_error("conv_plan_options.struct_size is %d, expected %d (use conv_plan_options_init)", o->struct_size,
                     (int)sizeof(conv_plan_options));
        return CONV_ERR_INVALID_ARG;
    }
    if (o->gemm < CONV_GEMM_AUTO || o->gemm > CONV_GEMM_TCGEN05_F16X3) {
        fc_set_error("unknown gemm implementation %d", (int)o->gemm);
        return CONV_ERR_INVALID_ARG;
    }
    if (o->gauss_combine < -1 || o->gauss_combine > 1 || o->complex_mode < -1 || o->complex_mode > 1 ||
        o->chunk_images < 0 || o->generic_transforms < 0 || o->generic_transforms > 1 || o->single_cta_mma < 0 ||
        o->single_cta_mma > 1 || o->e2e_chunks < 0 || o->overlap_kernel_transform < -1 ||
        o->overlap_kernel_transform > 1 || o->fused < 0 || o->fused > 1) {
        fc_set_error("conv_plan_options field out of range");
        return CONV_ERR_INVALID_ARG;
    }
    return CONV_OK;
}

// ---------------------------------------------------------------------------
// Tile-size planner: the paper's running-time model -- each stage
// bound by its compute or its memory traffic, stages summed -- with B200's
// measured HBM bandwidth and the contraction mode's tensor ceiling (MEASURED_PEAKS.json:
// 6534.5 GB/s, dense fp16/bf16 1634 TFLOP/s -> F16X3 545 and 3xTF32 272 fp32-equivalent
// TFLOP/s, three products per fp32 product; FFMA 74 TFLOP/s = 148 SMs x 128 lanes x 2 x
// 1.965 GHz).  Each stage's time is divided by the fraction of its roofline this kernel
// family reaches on B200 (kModelEff, measured over BASELINE.json's configs; DESIGN.md
// section 7), and the contraction's tensor work counts the padded columns it really issues.
// ---------------------------------------------------------------------------
namespace {
// Fraction of each stage's roofline the B200 kernels reach, measured over BASELINE.json's
// configs with L2 flushed between steps (profiles/r02_autotune_flushed_configs.json):
// the Winograd transforms 0.8-0.9; the FFT transforms depend on the tile edge t (codelet
// radices, and the per-tile state -- t complex values per thread, m x h staged spectra per
// tile -- that bounds the resident warps for large t); NK1 ~0.45;
// NK3 ~0.85 of max(tensor, HBM).
struct ModelEff {
    double nk1, nk2, nk3, nk4;
};
ModelEff model_eff(int method, int t) {
    // NK2 / NK4 per tile edge t (mean of VGG-1.2 and VGG-3.2, r02 flushed sweep)
    struct TE {
        int t;
        double nk2, nk4;
    };
    static const TE wino[] = {{4, 0.81, 0.78}, {5, 0.78, 0.85}, {6, 0.93, 0.92}, {8, 0.84, 0.78}};
    static const TE fft[] = {{4, 0.55, 0.42},  {5, 0.58, 0.45},  {6, 0.62, 0.55},  {7, 0.60, 0.50},
                             {8, 0.70, 0.62},  {9, 0.70, 0.58},  {10, 0.68, 0.58}, {12, 0.72, 0.59},
                             {13, 0.62, 0.56}, {14, 0.74, 0.57}, {15, 0.65, 0.53}, {16, 0.80, 0.67},
                             {18, 0.60, 0.52}, {20, 0.63, 0.52}, {21, 0.53, 0.37}, {24, 0.58, 0.47},
                             {25, 0.48, 0.41}, {27, 0.50, 0.43}, {28, 0.55, 0.35}, {30, 0.50, 0.42},
                             {31, 0.30, 0.33}, {32, 0.42, 0.39}};
    const bool w = method == CONV_WINOGRAD;
    const TE *tab = w ? wino : fft;
    const int n = w ? 4 : 22;
    ModelEff e = {w ? 0.50 : 0.45, w ? 0.85 : 0.55, 0.85, w ? 0.85 : 0.45};
    for (int i = 0; i < n; ++i)
        if (tab[i].t == t) {
            e.nk2 = tab[i].nk2;
            e.nk4 = tab[i].nk4;
        }
    return e;
}
}  // namespace

double fc_model_ms(const conv_plan_info &I, const Geometry &G) {
    const double bw = 6534.5e9;
    const int gemm = I.gemm;
    const double peak = gemm == CONV_GEMM_TCGEN05_F16X3 ? 1634.2e12 / 3.0
                        : gemm == CONV_GEMM_TCGEN05_3XTF32 ? 0.5 * 1634.2e12 / 3.0 : 74.4e12;
    const ModelEff ef = model_eff(G.method, G.t);
    const double eff[4] = {ef.nk1, ef.nk2, ef.nk3, ef.nk4};
    double t = 0.0;
    for (int s = 0; s < 4; ++s) {
        double ts = I.alg_bytes[s] / bw;
        if (s == 2) {  // tensor work on the padded columns (N = 128 / 256 tiles)
            const double pad = I.BN > 0 ? (double)I.BN_pad / (double)I.BN : 1.0;
            ts = std::max(ts, I.alg_flops[2] * pad / peak);
        }
        t += ts / eff[s];
    }
    return t * 1e3;
}

conv_status fc_best_m(int B, int C, int Cout, int H, int W, int r, int method, const conv_plan_options *opts,
                      int *m_out, double *model_ms, int max_cand, int *n_cand, int *cand_m, double *cand_ms) {
    if (method != CONV_WINOGRAD && method != CONV_REGULAR_FFT && method != CONV_GAUSS_FFT) {
        fc_set_error("conv_plan_best_m: method %d has no tile size", method);
        return CONV_ERR_INVALID_ARG;
    }
    const int tmax = method == CONV_WINOGRAD ? 8 : 32;
    int best = 0, nc = 0;
    double best_t = 0.0;
    conv_status last = CONV_ERR_UNSUPPORTED;
    for (int m = 1; m + r - 1 <= tmax; ++m) {
        if (!fc_fast_transforms(method, m + r - 1, m, r)) continue;
        Geometry g;
        conv_plan_info I;
        conv_status st = fc_fill_geometry(B, C, Cout, H, W, r, method, m, &g, &I, opts);
        if (st != CONV_OK) {
            last = st;
            continue;
        }
        if (I.gemm == CONV_GEMM_AUTO) I.gemm = CONV_GEMM_TCGEN05_F16X3;
        const double t = fc_model_ms(I, g);
        if (cand_m && cand_ms && nc < max_cand) {
            cand_m[nc] = m;
            cand_ms[nc] = t;
        }
        ++nc;
        if (!best || t < best_t) {  // strict: ties keep the smaller m
            best = m;
            best_t = t;
        }
    }
    if (n_cand) *n_cand = nc < max_cand ? nc : max_cand;
    if (!best) {
        if (last == CONV_ERR_UNSUPPORTED)
            fc_set_error("conv_plan_best_m: no compiled tile size for method %d with r = %d", method, r);
        return last;
    }
    *m_out = best;
    if (model_ms) *model_ms = best_t;
    return CONV_OK;
}

// The part of the plan shared by 2-D and N-D layers: contraction shape (Z, M, K, Kp,
// complex mode, Gauss combine) and the info block (workspace sizes, algorithmic bytes and
// FLOPs of Table layer-stuff P:1025-1032 with c = C, c' = C', alpha = 1, generalised to
// volumes: prod in_d, prod r_d, prod o_d).  G: B, C, Cout, method, t / E / N / BN(_pad),
// planes, vin, vout, kvol, (nd axes) filled.
static conv_status finish_geometry(Geometry &G, conv_plan_info *info, const conv_plan_options *opts) {
    const conv_gemm_impl gemm = opts->gemm;
    const int method = G.method, B = G.B, C = G.C, Cout = G.Cout;
    if (method != CONV_DIRECT) {
        G.divN = fc_fastdiv(G.N);
        G.divNw = fc_fastdiv(G.n_w > 0 ? G.n_w : 1);
        G.BN = (long long)B * G.N;
        G.BN_pad = (G.BN + FC_TB - 1) / FC_TB * FC_TB;
        if (G.BN >= (1LL << 31)) {
            fc_set_error("too many tiles (B N = %lld)", G.BN);
            return CONV_ERR_UNSUPPORTED;
        }
        if (method == CONV_REGULAR_FFT) {  // real embedding of the complex product
            G.Z = G.E; G.M = 2 * Cout; G.K = 2 * C;
        } else if (method == CONV_GAUSS_FFT) {
            G.Z = 3 * G.E; G.M = Cout; G.K = C;
        } else {
            G.Z = G.E; G.M = Cout; G.K = C;
        }
        G.fused = opts->fused == 1;
        if (G.fused && (method != CONV_WINOGRAD || G.m != 2 || G.r != 3 || G.nd != 0 || opts->chunk_images != 0 ||
                        (gemm != CONV_GEMM_AUTO && gemm != CONV_GEMM_TCGEN05_3XTF32))) {
            fc_set_error("fused NK2-NK4 needs 2-D Winograd F(2,3), the 3xTF32 contraction (gemm AUTO or "
                         "TCGEN05_3XTF32) and chunk_images 0");
            return CONV_ERR_UNSUPPORTED;
        }
        // AUTO: query-time default F16X3 (fused plans: 3xTF32)
        G.vf16 = !G.fused && (gemm == CONV_GEMM_TCGEN05_F16X3 || gemm == CONV_GEMM_AUTO);
        const int kq = G.vf16 ? 8 : 4;  // V row pitch: 16 bytes of fp16 / fp32
        G.Kp = (G.K + kq - 1) / kq * kq;
        G.gc = method == CONV_GAUSS_FFT && G.vf16 && Cout % 32 == 0 && gauss_combine_pays(G, opts->gauss_combine);
        G.Xz = G.gc ? G.E : G.Z;
        G.Xm = G.gc ? 2 * Cout : G.M;
        G.cplx = 0;
        if (method == CONV_REGULAR_FFT && gemm != CONV_GEMM_FFMA && Cout % 256 == 0 && C % (G.vf16 ? 32 : 16) == 0 &&
            opts->complex_mode != 0) {
            G.cplx = 1;
            G.Kp = (C + kq - 1) / kq * kq;
        }
    }
    G.tc_1sm = opts->single_cta_mma;
    G.e_lo = 0;
    G.e_hi = G.E;
    if (!info) return CONV_OK;
    conv_plan_info I;
    memset(&I, 0, sizeof(I));
    I.B = B; I.C = C; I.Cout = Cout; I.H = G.H; I.W = G.W; I.r = G.r; I.m = G.m; I.method = method;
    I.Ho = G.Ho; I.Wo = G.Wo; I.t = G.t; I.n_h = G.n_h; I.n_w = G.n_w; I.N = G.N; I.h = G.h;
    I.E = G.E; I.planes = G.planes; I.BN = G.BN; I.BN_pad = G.BN_pad;
    I.gemm_Z = G.Z; I.gemm_M = G.M; I.gemm_K = G.K;
    I.nd = G.nd ? G.nd : 2;
    for (int d = 0; d < 3; ++d) {
        I.in_shape[d] = G.ax_in[d]; I.kernel_shape[d] = G.ax_r[d]; I.m_shape[d] = G.ax_m[d];
        I.t_shape[d] = G.ax_t[d]; I.tiles[d] = G.ax_n[d]; I.out_shape[d] = G.ax_o[d];
    }
    const double vin = (double)G.vin, vout = (double)G.vout, kv = (double)G.kvol;
    I.direct_flops = 2.0 * B * (double)C * Cout * vout * kv;
    I.chunk = B;
    I.nchunks = 1;
    I.gemm = gemm == CONV_GEMM_AUTO ? (G.fused ? CONV_GEMM_TCGEN05_3XTF32 : CONV_GEMM_TCGEN05_F16X3) : gemm;
    I.fused = G.fused;
    I.x_planes = method == CONV_DIRECT ? 0 : (G.gc ? 2 : G.planes);
    if (method != CONV_DIRECT) {
        const int split = (gemm != CONV_GEMM_FFMA);
        const size_t vb = fc_v_bytes(G);  // V_hi, then V_lo at the next 256 B boundary
        I.bytes_V = split ? align256(vb) + vb : vb;
        I.chunk = pick_chunk(G, opts->chunk_images);
        if (G.vf16)  // + per-c' scales [2][C'] and the per-image max|U_b| words of a chunk
            I.bytes_V = align256(I.bytes_V) + align256((size_t)2 * Cout * 4) + align256((size_t)I.chunk * 4);
        I.nchunks = (B + I.chunk - 1) / I.chunk;
        const Geometry Gc = fc_chunk_geometry(G, I.chunk);
        I.BN_pad = Gc.BN_pad;
        I.bytes_U = (size_t)G.Z * G.K * Gc.BN_pad * 4;
        I.bytes_X = (size_t)G.Xz * G.Xm * Gc.BN_pad * 4;
        I.workspace_bytes = align256(I.bytes_V) + align256(I.bytes_U) + align256(I.bytes_X);
        const double BCN = (double)B * C * G.N, BCpN = (double)B * Cout * G.N;
        const double CCp = (double)C * Cout;
        const double BN = (double)B * G.N;
        // reals per transformed tile: wE = E (Winograd), 2E (Regular), 3E (Gauss)
        const double wEr = method == CONV_GAUSS_FFT ? 3.0 * G.E : (method == CONV_REGULAR_FFT ? 2.0 * G.E : (double)G.E);
        I.alg_bytes[0] = 4.0 * CCp * kv + 4.0 * wEr * CCp;
        I.alg_bytes[1] = 4.0 * B * C * vin + 4.0 * wEr * BCN;
        // X carries x_planes real planes per element (Gauss combined in NK3's epilogue: 2)
        const double wX = G.gc ? 2.0 * G.E : wEr;
        I.alg_bytes[2] = 4.0 * wEr * (BN * C + CCp) + 4.0 * wX * BN * Cout;
        I.alg_bytes[3] = 4.0 * wX * BCpN + 4.0 * B * Cout * vout;
        // element-wise FLOPs: 2t^2 BNCC' / 8 t h BNCC' / 6 t h BNCC'
        const double k = method == CONV_WINOGRAD ? 2.0 : (method == CONV_REGULAR_FFT ? 8.0 : 6.0);
        I.alg_flops[2] = k * G.E * BN * CCp;
        if (G.fused) {  // one kernel: input + V (hi, lo) + output; no U / X in the workspace
            I.bytes_U = I.bytes_X = 0;
            I.workspace_bytes = align256(I.bytes_V);
            I.alg_bytes[2] = 4.0 * B * C * vin + 4.0 * wEr * CCp + 4.0 * B * Cout * vout;
            I.alg_bytes[1] = I.alg_bytes[3] = 0.0;
            I.x_planes = 0;
        }
    } else {
        I.alg_bytes[2] = 4.0 * B * C * vin + 4.0 * Cout * C * kv + 4.0 * B * Cout * vout;
        I.alg_flops[2] = I.direct_flops;
    }
    *info = I;
    return CONV_OK;
}

conv_status fc_fill_geometry(int B, int C, int Cout, int H, int W, int r, int method, int m,
                             Geometry *g, conv_plan_info *info, const conv_plan_options *opts) {
    {
        conv_status st = check_options(opts);
        if (st != CONV_OK) return st;
    }
    if (B < 1 || C < 1 || Cout < 1 || H < 1 || W < 1 || r < 1) {
        fc_set_error("sizes must be >= 1 (B=%d C=%d C'=%d H=%d W=%d r=%d)", B, C, Cout, H, W, r);
        return CONV_ERR_INVALID_ARG;
    }
    if (H < r || W < r) {
        fc_set_error("image %dx%d smaller than kernel %d", H, W, r);
        return CONV_ERR_INVALID_ARG;
    }
    if (method < CONV_DIRECT || method > CONV_GAUSS_FFT) {
        fc_set_error("unknown method %d", method);
        return CONV_ERR_INVALID_ARG;
    }
    if (method != CONV_DIRECT && m < 0) {
        fc_set_error("output tile m must be >= 1, or 0 for the planner's choice (got %d)", m);
        return CONV_ERR_INVALID_ARG;
    }
    if (method != CONV_DIRECT && m == 0) {  // the planner's tile (conv_plan_best_m)
        conv_status st = fc_best_m(B, C, Cout, H, W, r, method, opts, &m, nullptr, 0, nullptr, nullptr, nullptr);
        if (st != CONV_OK) return st;
    }
    if ((long long)B * C * H * W >= (1LL << 40) || (long long)Cout * C * r * r >= (1LL << 40)) {
        fc_set_error("tensor too large");
        return CONV_ERR_UNSUPPORTED;
    }
    Geometry G = {};
    G.B = B; G.C = C; G.Cout = Cout; G.H = H; G.W = W; G.r = r; G.method = method;
    G.Ho = H - r + 1;
    G.Wo = W - r + 1;
    G.nd = 0;
    G.vin = (long long)H * W;
    G.vout = (long long)G.Ho * G.Wo;
    G.kvol = r * r;
    G.ax_in[0] = 1; G.ax_in[1] = H; G.ax_in[2] = W;
    G.ax_r[0] = 1; G.ax_r[1] = r; G.ax_r[2] = r;
    G.ax_o[0] = 1; G.ax_o[1] = G.Ho; G.ax_o[2] = G.Wo;
    G.ax_m[0] = G.ax_t[0] = G.ax_n[0] = G.ax_len[0] = 1;
    if (method == CONV_DIRECT) {
        G.m = 0;
    } else {
        G.m = m;
        G.t = m + r - 1;
        if (method == CONV_WINOGRAD) {
            if (r < 2 || m < 2 || G.t > 8) {
                fc_set_error("Winograd F(%d,%d) unsupported: need r>=2, m>=2, t<=8 (t=%d)", m, r, G.t);
                return CONV_ERR_UNSUPPORTED;
            }
            G.h = G.t;
            G.planes = 1;
        } else {
            if (G.t > FC_MAX_T) {
                fc_set_error("FFT tile t=%d exceeds %d", G.t, FC_MAX_T);
                return CONV_ERR_UNSUPPORTED;
            }
            G.h = G.t / 2 + 1;  // == ceil((t+1)/2)
            G.planes = method == CONV_REGULAR_FFT ? 2 : 3;
        }
        G.n_h = (G.Ho + m - 1) / m;
        G.n_w = (G.Wo + m - 1) / m;
        G.N = G.n_h * G.n_w;
        G.E = G.t * G.h;
        G.ax_m[1] = G.ax_m[2] = m;
        G.ax_t[1] = G.ax_t[2] = G.t;
        G.ax_n[1] = G.n_h; G.ax_n[2] = G.n_w;
        G.ax_len[1] = G.t; G.ax_len[2] = G.h;
    }
    conv_status st = finish_geometry(G, info, opts);
    if (st != CONV_OK) return st;
    *g = G;
    return CONV_OK;
}

// N-dimensional / non-isotropic geometry (conv_plan_nd): per-axis sizes right-aligned in 3
// slots.  nd == 2 with a square kernel and equal tiles is the 2-D isotropic plan (fast path).
conv_status fc_fill_geometry_nd(int nd, int B, int C, int Cout, const int *in, const int *rk, int method,
                                const int *mt, Geometry *g, conv_plan_info *info, const conv_plan_options *opts) {
    conv_status st = check_options(opts);
    if (st != CONV_OK) return st;
    if (nd < 1 || nd > 3 || !in || !rk || (method != CONV_DIRECT && !mt)) {
        fc_set_error("conv_plan_nd: nd must be 1..3 and the shape arrays non-NULL");
        return CONV_ERR_INVALID_ARG;
    }
    if (method < CONV_DIRECT || method > CONV_GAUSS_FFT) {
        fc_set_error("unknown method %d", method);
        return CONV_ERR_INVALID_ARG;
    }
    if (nd == 2 && rk[0] == rk[1] && (method == CONV_DIRECT || (mt[0] == mt[1] && mt[0] > 0)))
        return fc_fill_geometry(B, C, Cout, in[0], in[1], rk[0], method, method == CONV_DIRECT ? 0 : mt[0], g, info,
                                opts);
    if (B < 1 || C < 1 || Cout < 1) {
        fc_set_error("sizes must be >= 1 (B=%d C=%d C'=%d)", B, C, Cout);
        return CONV_ERR_INVALID_ARG;
    }
    Geometry G = {};
    G.B = B; G.C = C; G.Cout = Cout; G.method = method; G.nd = nd;
    G.vin = G.vout = 1;
    G.kvol = 1;
    long long ntile = 1, E = 1;
    int tmax = 1;
    for (int d = 0; d < 3; ++d) {
        G.ax_in[d] = G.ax_r[d] = G.ax_m[d] = G.ax_t[d] = G.ax_n[d] = G.ax_o[d] = G.ax_len[d] = 1;
    }
    for (int i = 0; i < nd; ++i) {
        const int d = 3 - nd + i;
        if (in[i] < 1 || rk[i] < 1 || in[i] < rk[i]) {
            fc_set_error("axis %d: input %d and kernel %d must be >= 1 with input >= kernel", i, in[i], rk[i]);
            return CONV_ERR_INVALID_ARG;
        }
        G.ax_in[d] = in[i];
        G.ax_r[d] = rk[i];
        G.ax_o[d] = in[i] - rk[i] + 1;
        G.vin *= in[i];
        G.vout *= G.ax_o[d];
        G.kvol *= rk[i];
        if (method == CONV_DIRECT) continue;
        if (mt[i] < 1) {
            fc_set_error("axis %d: output tile m must be >= 1 (got %d)", i, mt[i]);
            return CONV_ERR_INVALID_ARG;
        }
        G.ax_m[d] = mt[i];
        G.ax_t[d] = mt[i] + rk[i] - 1;
        if (method == CONV_WINOGRAD) {
            if (rk[i] > 1 && (mt[i] < 2 || G.ax_t[d] > 8)) {
                fc_set_error("axis %d: Winograd F(%d,%d) unsupported: need m>=2, t<=8 (r = 1 axes: any m)", i, mt[i],
                             rk[i]);
                return CONV_ERR_UNSUPPORTED;
            }
            if (rk[i] == 1 && mt[i] > 8) {
                fc_set_error("axis %d: Winograd tile %d exceeds 8", i, mt[i]);
                return CONV_ERR_UNSUPPORTED;
            }
        } else if (G.ax_t[d] > FC_MAX_T) {
            fc_set_error("axis %d: FFT tile t=%d exceeds %d", i, G.ax_t[d], FC_MAX_T);
            return CONV_ERR_UNSUPPORTED;
        }
        G.ax_n[d] = (G.ax_o[d] + mt[i] - 1) / mt[i];
        G.ax_len[d] = (method != CONV_WINOGRAD && i == nd - 1) ? G.ax_t[d] / 2 + 1 : G.ax_t[d];
        ntile *= G.ax_n[d];
        E *= G.ax_len[d];
        tmax = G.ax_t[d] > tmax ? G.ax_t[d] : tmax;
    }
    if ((long long)B * C * G.vin >= (1LL << 40) || (long long)Cout * C * G.kvol >= (1LL << 40) ||
        (long long)B * Cout * G.vout >= (1LL << 40) || ntile >= (1LL << 31) || E >= (1LL << 20)) {
        fc_set_error("tensor too large");
        return CONV_ERR_UNSUPPORTED;
    }
    // 2-D-style fields for reporting (the last two axes)
    G.H = G.ax_in[1]; G.W = G.ax_in[2]; G.Ho = G.ax_o[1]; G.Wo = G.ax_o[2];
    G.r = G.ax_r[2];
    if (method == CONV_DIRECT) {
        G.m = 0;
    } else {
        G.m = G.ax_m[2];
        G.t = G.ax_t[2];
        G.h = G.ax_len[2];
        G.n_h = G.ax_n[1];
        G.n_w = G.ax_n[2];
        G.N = (int)ntile;
        G.E = (int)E;
        G.planes = method == CONV_WINOGRAD ? 1 : (method == CONV_REGULAR_FFT ? 2 : 3);
        const long long vt = (long long)G.ax_t[0] * G.ax_t[1] * G.ax_t[2];
        if (vt * 16 > 200 * 1024) {
            fc_set_error("N-D tile volume %lld too large for the generic transforms", vt);
            return CONV_ERR_UNSUPPORTED;
        }
    }
    (void)tmax;
    st = finish_geometry(G, info, opts);
    if (st != CONV_OK) return st;
    *g = G;
    return CONV_OK;
}

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
extern "C" {

const char *conv_status_string(conv_status s) {
    switch (s) {
        case CONV_OK: return "CONV_OK";
        case CONV_ERR_INVALID_ARG: return "CONV_ERR_INVALID_ARG";
        case CONV_ERR_UNSUPPORTED: return "CONV_ERR_UNSUPPORTED";
        case CONV_ERR_OUT_OF_MEMORY: return "CONV_ERR_OUT_OF_MEMORY";
        case CONV_ERR_CUDA: return "CONV_ERR_CUDA";
        case CONV_ERR_DEVICE_MISMATCH: return "CONV_ERR_DEVICE_MISMATCH";
    }
    return "CONV_ERR_UNKNOWN";
}

const char *conv_last_error(void) { return g_err; }

void conv_plan_options_init(conv_plan_options *o) {
    if (!o) return;
    memset(o, 0, sizeof(*o));
    o->struct_size = (int)sizeof(conv_plan_options);
    o->gemm = CONV_GEMM_AUTO;
    o->gauss_combine = -1;
    o->complex_mode = -1;
    o->chunk_images = 0;
    o->generic_transforms = 0;
    o->single_cta_mma = 0;
    o->e2e_chunks = 0;
    o->overlap_kernel_transform = -1;
    o->fused = 0;
}

static const conv_plan_options *opts_or_default(const conv_plan_options *o, conv_plan_options *tmp) {
    if (o) return o;
    conv_plan_options_init(tmp);
    return tmp;
}

conv_status conv_plan_query_opts(int B, int C, int Cout, int H, int W, int r, conv_method method, int m,
                                 const conv_plan_options *opts, conv_plan_info *info) {
    conv_plan_options d;
    Geometry g;
    return fc_fill_geometry(B, C, Cout, H, W, r, (int)method, m, &g, info, opts_or_default(opts, &d));
}

conv_status conv_plan_query(int B, int C, int Cout, int H, int W, int r, conv_method method, int m,
                            conv_plan_info *info) {
    return conv_plan_query_opts(B, C, Cout, H, W, r, method, m, nullptr, info);
}

conv_status conv_plan_best_method(int B, int C, int Cout, int H, int W, int r, const conv_plan_options *opts,
                                  conv_method *method_out, int *m_out, double *model_ms) {
    if (!method_out || !m_out) {
        fc_set_error("conv_plan_best_method: NULL output");
        return CONV_ERR_INVALID_ARG;
    }
    conv_plan_options d;
    const conv_plan_options *o = opts_or_default(opts, &d);
    int best_m = 0;
    double best = 0.0;
    conv_method best_meth = CONV_DIRECT;
    conv_status last = CONV_ERR_UNSUPPORTED;
    const conv_method order[3] = {CONV_WINOGRAD, CONV_REGULAR_FFT, CONV_GAUSS_FFT};
    for (conv_method meth : order) {
        int m = 0;
        double ms = 0.0;
        conv_status st = fc_best_m(B, C, Cout, H, W, r, (int)meth, o, &m, &ms, 0, nullptr, nullptr, nullptr);
        if (st != CONV_OK) {
            last = st;
            continue;
        }
        if (!best_m || ms < best) {  // the paper's rule: each method at its best m, the fastest wins
            best_m = m;
            best = ms;
            best_meth = meth;
        }
    }
    if (!best_m) return last;
    *method_out = best_meth;
    *m_out = best_m;
    if (model_ms) *model_ms = best;
    return CONV_OK;
}

conv_status conv_plan_best_m(int B, int C, int Cout, int H, int W, int r, conv_method method,
                             const conv_plan_options *opts, int *m_out, double *model_ms, int max_cand, int *n_cand,
                             int *cand_m, double *cand_ms) {
    if (!m_out || max_cand < 0) {
        fc_set_error("conv_plan_best_m: NULL m_out or negative max_cand");
        return CONV_ERR_INVALID_ARG;
    }
    conv_plan_options d;
    return fc_best_m(B, C, Cout, H, W, r, (int)method, opts_or_default(opts, &d), m_out, model_ms, max_cand, n_cand,
                     cand_m, cand_ms);
}

conv_status conv_winograd_matrices(int m, int r, double *AT, double *BT, double *G) {
    if (!AT || !BT || !G) {
        fc_set_error("NULL output pointer");
        return CONV_ERR_INVALID_ARG;
    }
    return fc_winograd_rational(m, r, AT, BT, G);
}

// nd = 0: the 2-D isotropic plan (H, W, r, m); nd = 1..3: conv_plan_nd's shapes (in, rk, mt)
static conv_status plan_create(conv_plan_t *out, int nd, int B, int C, int Cout, int H, int W, int r,
                               conv_method method, int m, const int *in, const int *rk, const int *mt,
                               const conv_plan_options *opts_in) {
    if (!out) {
        fc_set_error("NULL plan pointer");
        return CONV_ERR_INVALID_ARG;
    }
    conv_plan_options opts;
    if (opts_in) {
        conv_status st = check_options(opts_in);
        if (st != CONV_OK) return st;
        opts = *opts_in;
    } else {
        conv_plan_options_init(&opts);
    }
    conv_plan_s *p = (conv_plan_s *)calloc(1, sizeof(conv_plan_s));
    if (!p) return CONV_ERR_OUT_OF_MEMORY;
    conv_gemm_impl gemm = opts.gemm;
    if (gemm == CONV_GEMM_AUTO)
        gemm = !fc_tcgen05_available() ? CONV_GEMM_FFMA
                                       : (opts.fused == 1 ? CONV_GEMM_TCGEN05_3XTF32 : CONV_GEMM_TCGEN05_F16X3);
    if ((gemm == CONV_GEMM_TCGEN05_3XTF32 || gemm == CONV_GEMM_TCGEN05_F16X3) && !fc_tcgen05_available()) {
        free(p);
        fc_set_error("tcgen05 contraction not available in this build");
        return CONV_ERR_UNSUPPORTED;
    }
    opts.gemm = gemm;
    conv_status st = nd == 0 ? fc_fill_geometry(B, C, Cout, H, W, r, (int)method, m, &p->g, &p->info, &opts)
                             : fc_fill_geometry_nd(nd, B, C, Cout, in, rk, (int)method, mt, &p->g, &p->info, &opts);
    if (st != CONV_OK) { free(p); return st; }
    p->gemm = gemm;
    const Geometry &g = p->g;
    ConvConsts &cc = p->host_consts;
    memset(&cc, 0, sizeof(cc));
    NdConsts ndc;
    memset(&ndc, 0, sizeof(ndc));
    if (g.nd && method != CONV_DIRECT) {
        // per-axis constants (exact rationals / fp64 twiddles, rounded once) and the F16X3 bound
        // |V| <= prod_d (max_k sum_p |G_d[k][p]|) max|g|  (FFT: prod r_d / prod t_d, x2 Gauss)
        double bound = method == CONV_GAUSS_FFT ? 2.0 : 1.0;
        for (int d = 3 - g.nd; d < 3; ++d) {
            const int md = g.ax_m[d], rd = g.ax_r[d], td = g.ax_t[d];
            if (method == CONV_WINOGRAD) {
                double at[64], bt[64], gm[64];
                if (rd == 1) {  // F(m, 1): identity transforms, G = ones
                    for (int i = 0; i < 64; ++i) at[i] = bt[i] = gm[i] = 0.0;
                    for (int i = 0; i < td; ++i) {
                        at[i * td + i] = bt[i * td + i] = 1.0;
                        gm[i] = 1.0;
                    }
                } else {
                    st = fc_winograd_rational(md, rd, at, bt, gm);
                    if (st != CONV_OK) { free(p); return st; }
                }
                for (int i = 0; i < td * td; ++i) ndc.BT[d][i] = (float)bt[i];
                for (int i = 0; i < td * rd; ++i) ndc.G[d][i] = (float)gm[i];
                for (int i = 0; i < md * td; ++i) ndc.AT[d][i] = (float)at[i];
                double rs = 0.0;
                for (int k = 0; k < td; ++k) {
                    double a_ = 0.0;
                    for (int q = 0; q < rd; ++q) a_ += fabs(gm[k * rd + q]);
                    rs = a_ > rs ? a_ : rs;
                }
                bound *= rs;
            } else {
                for (int j = 0; j < td; ++j) {
                    const double ang = 2.0 * M_PI * (double)j / (double)td;
                    ndc.cosv[d][j] = (float)cos(ang);
                    ndc.sinv[d][j] = (float)sin(ang);
                }
                bound *= (double)rd / (double)td;
            }
        }
        p->g.vbound = (float)bound;
    } else if (method == CONV_WINOGRAD) {
        st = fc_winograd_rational(g.m, g.r, p->AT64, p->BT64, p->G64);
        if (st != CONV_OK) { free(p); return st; }
        for (int i = 0; i < g.t * g.t; ++i) cc.BT[i] = (float)p->BT64[i];
        for (int i = 0; i < g.t * g.r; ++i) cc.G[i] = (float)p->G64[i];
        for (int i = 0; i < g.m * g.t; ++i) cc.AT[i] = (float)p->AT64[i];
        // |V[k][l]| = |sum_pq G[k][p] g[p][q] G[l][q]| <= (max_k sum_p |G[k][p]|)^2 max|g|
        double rs = 0.0;
        for (int k = 0; k < g.t; ++k) {
            double a = 0.0;
            for (int q = 0; q < g.r; ++q) a += fabs(p->G64[k * g.r + q]);
            rs = a > rs ? a : rs;
        }
        p->g.vbound = (float)(rs * rs);
    } else if (method != CONV_DIRECT) {
        // |DFT2(pad g)| / t^2 <= r^2 max|g| / t^2; Gauss planes V_i -+ V_r at most twice that
        p->g.vbound = (float)((method == CONV_GAUSS_FFT ? 2.0 : 1.0) * g.r * g.r / ((double)g.t * g.t));
        for (int j = 0; j < g.t; ++j) {  // twiddles in fp64, rounded once (reading R11)
            const double ang = 2.0 * M_PI * (double)j / (double)g.t;
            cc.cosv[j] = (float)cos(ang);
            cc.sinv[j] = (float)sin(ang);
        }
    }
    p->generic_transforms = opts.generic_transforms;
    cudaError_t e = cudaGetDevice(&p->device);
    if (e != cudaSuccess) {
        fc_set_error("cudaGetDevice: %s", cudaGetErrorString(e));
        free(p);
        return CONV_ERR_CUDA;
    }
    {  // the library carries sm_100a code only (no PTX): refuse other devices up front
        int major = 0, minor = 0;
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, p->device);
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, p->device);
        if (major != 10 || minor != 0) {
            fc_set_error("device %d is sm_%d%d; this build targets sm_100a (B200) only", p->device, major, minor);
            free(p);
            return CONV_ERR_UNSUPPORTED;
        }
    }
    if (method != CONV_DIRECT) {
        if (method != CONV_WINOGRAD && (e = fc_init_twiddles()) != cudaSuccess) {
            fc_set_error("twiddle upload: %s", cudaGetErrorString(e));
            free(p);
            return CONV_ERR_CUDA;
        }
        e = cudaMalloc(&p->d_consts, sizeof(ConvConsts));
        if (e != cudaSuccess) {
            fc_set_error("cudaMalloc(consts): %s", cudaGetErrorString(e));
            free(p);
            return e == cudaErrorMemoryAllocation ? CONV_ERR_OUT_OF_MEMORY : CONV_ERR_CUDA;
        }
        e = cudaMemcpy(p->d_consts, &cc, sizeof(ConvConsts), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            fc_set_error("cudaMemcpy(consts): %s", cudaGetErrorString(e));
            cudaFree(p->d_consts);
            free(p);
            return CONV_ERR_CUDA;
        }
        if (g.nd) {
            e = cudaMalloc(&p->d_nd, sizeof(NdConsts));
            if (e == cudaSuccess) e = cudaMemcpy(p->d_nd, &ndc, sizeof(NdConsts), cudaMemcpyHostToDevice);
            if (e != cudaSuccess) {
                fc_set_error("N-D constants: %s", cudaGetErrorString(e));
                if (p->d_nd) cudaFree(p->d_nd);
        if (p->aux) cudaStreamDestroy(p->aux);
        for (int i = 0; i < FC_EVPAIRS; ++i) {
            if (p->fork_ev[i]) cudaEventDestroy(p->fork_ev[i]);
            if (p->join_ev[i]) cudaEventDestroy(p->join_ev[i]);
        }
                cudaFree(p->d_consts);
                free(p);
                return e == cudaErrorMemoryAllocation ? CONV_ERR_OUT_OF_MEMORY : CONV_ERR_CUDA;
            }
        }
        p->off_V = 0;
        const size_t vb = fc_v_bytes(g);
        p->off_Vlo = align256(vb);
        if (g.vf16) {
            p->off_vscale = p->off_Vlo + align256(vb);
            p->off_umax = p->off_vscale + align256((size_t)2 * g.Cout * 4);
        }
        const size_t vtot = align256(p->info.bytes_V);
        p->off_U = vtot;
        p->off_X = vtot + align256(p->info.bytes_U);
        p->ws_bytes = p->info.workspace_bytes;
        if (gemm == CONV_GEMM_FFMA) p->off_Vlo = 0;
    }
    p->chunk = p->info.chunk;
    p->nchunks = p->info.nchunks;
    p->e2e_chunks = opts.e2e_chunks > 0 ? opts.e2e_chunks : 8;
    p->overlap_nk1 = opts.overlap_kernel_transform != 0 && method != CONV_DIRECT;
    if (p->overlap_nk1) {  // NK1 || NK2: an auxiliary stream and fork / join events
        bool ok = cudaStreamCreateWithFlags(&p->aux, cudaStreamNonBlocking) == cudaSuccess;
        for (int i = 0; ok && i < FC_EVPAIRS; ++i)
            ok = cudaEventCreateWithFlags(&p->fork_ev[i], cudaEventDisableTiming) == cudaSuccess &&
                 cudaEventCreateWithFlags(&p->join_ev[i], cudaEventDisableTiming) == cudaSuccess;
        if (!ok) {  // fall back to the serial order
            cudaGetLastError();
            p->overlap_nk1 = 0;
        }
    }
    // the pipelined host path's copy streams are created on its first call (conv_forward_host)
    *out = p;
    return CONV_OK;
}

conv_status conv_plan_opts(conv_plan_t *out, int B, int C, int Cout, int H, int W, int r,
                           conv_method method, int m, const conv_plan_options *opts) {
    return plan_create(out, 0, B, C, Cout, H, W, r, method, m, nullptr, nullptr, nullptr, opts);
}

conv_status conv_plan_nd(conv_plan_t *out, int nd, int B, int C, int Cout, const int *in_shape,
                         const int *kernel_shape, conv_method method, const int *m, const conv_plan_options *opts) {
    return plan_create(out, nd, B, C, Cout, 0, 0, 0, method, 0, in_shape, kernel_shape, m, opts);
}

conv_status conv_plan_query_nd(int nd, int B, int C, int Cout, const int *in_shape, const int *kernel_shape,
                               conv_method method, const int *m, const conv_plan_options *opts,
                               conv_plan_info *info) {
    conv_plan_options d;
    Geometry g;
    return fc_fill_geometry_nd(nd, B, C, Cout, in_shape, kernel_shape, (int)method, m, &g, info,
                               opts_or_default(opts, &d));
}

conv_status conv_plan_ex(conv_plan_t *out, int B, int C, int Cout, int H, int W, int r,
                         conv_method method, int m, conv_gemm_impl gemm) {
    conv_plan_options o;
    conv_plan_options_init(&o);
    o.gemm = gemm;
    return conv_plan_opts(out, B, C, Cout, H, W, r, method, m, &o);
}

conv_status conv_plan(conv_plan_t *out, int B, int C, int Cout, int H, int W, int r,
                      conv_method method, int m) {
    return conv_plan_opts(out, B, C, Cout, H, W, r, method, m, nullptr);
}

void conv_destroy(conv_plan_t p) {
    if (!p) return;
    if (p->inner) conv_destroy(p->inner);
    if (p->d_consts || p->d_nd || p->h2d || p->d2h || p->aux) {
        int cur = -1;
        cudaGetDevice(&cur);
        if (cur != p->device) cudaSetDevice(p->device);
        if (p->d_consts) cudaFree(p->d_consts);
        if (p->d_nd) cudaFree(p->d_nd);
        if (p->aux) cudaStreamDestroy(p->aux);
        for (int i = 0; i < FC_EVPAIRS; ++i) {
            if (p->fork_ev[i]) cudaEventDestroy(p->fork_ev[i]);
            if (p->join_ev[i]) cudaEventDestroy(p->join_ev[i]);
        }
        if (p->h2d) cudaStreamDestroy(p->h2d);
        if (p->d2h) cudaStreamDestroy(p->d2h);
        if (cur >= 0 && cur != p->device) cudaSetDevice(cur);
    }
    free(p);
}

conv_status conv_plan_get_info(conv_plan_t p, conv_plan_info *info) {
    if (!p || !info) {
        fc_set_error("NULL argument");
        return CONV_ERR_INVALID_ARG;
    }
    *info = p->info;
    return CONV_OK;
}

size_t conv_workspace_bytes(conv_plan_t p) { return p ? p->ws_bytes : 0; }

conv_status conv_workspace_layout(conv_plan_t p, size_t offsets[4]) {
    if (!p || !offsets) {
        fc_set_error("NULL argument");
        return CONV_ERR_INVALID_ARG;
    }
    offsets[0] = p->off_V;
    offsets[1] = p->off_Vlo;
    offsets[2] = p->off_U;
    offsets[3] = p->off_X;
    return CONV_OK;
}

conv_status conv_workspace_aux(conv_plan_t p, size_t offsets[2]) {
    if (!p || !offsets) {
        fc_set_error("NULL argument");
        return CONV_ERR_INVALID_ARG;
    }
    offsets[0] = p->off_vscale;
    offsets[1] = p->off_umax;
    return CONV_OK;
}

conv_status conv_plan_winograd_matrices(conv_plan_t p, double *AT, double *BT, double *G) {
    if (!p || !AT || !BT || !G) {
        fc_set_error("NULL argument");
        return CONV_ERR_INVALID_ARG;
    }
    if (p->g.method != CONV_WINOGRAD) {
        fc_set_error("not a Winograd plan");
        return CONV_ERR_UNSUPPORTED;
    }
    memcpy(AT, p->AT64, sizeof(double) * p->g.m * p->g.t);
    memcpy(BT, p->BT64, sizeof(double) * p->g.t * p->g.t);
    memcpy(G, p->G64, sizeof(double) * p->g.t * p->g.r);
    return CONV_OK;
}

int conv_forward_launch_count(conv_plan_t p) {
    if (!p) return 0;
    if (p->g.method == CONV_DIRECT) return 1;
    // F16X3 FFT plans run a per-c' scale prologue before the z-sliced FFT kernel transform
    const int nk1 = p->generic_transforms ? 1 : fc_nk1_launches(p->g, p->g.vf16 ? 2 : 1);
    return nk1 + 3 * p->nchunks;
}

// -- pointer checks ----------------------------------------------------------
static conv_status check_dev_ptr(const conv_plan_s *p, const void *ptr, const char *name) {
    if (!ptr) {
        fc_set_error("%s is NULL", name);
        return CONV_ERR_INVALID_ARG;
    }
    if (((uintptr_t)ptr) & 15) {
        fc_set_error("%s is not 16-byte aligned", name);
        return CONV_ERR_INVALID_ARG;
    }
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        fc_set_error("%s: cudaPointerGetAttributes: %s", name, cudaGetErrorString(e));
        return CONV_ERR_INVALID_ARG;
    }
    if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) {
        fc_set_error("%s is not device memory", name);
        return CONV_ERR_INVALID_ARG;
    }
    if (a.device != p->device) {
        fc_set_error("%s lives on device %d, plan on device %d", name, a.device, p->device);
        return CONV_ERR_DEVICE_MISMATCH;
    }
    return CONV_OK;
}

static conv_status check_device(const conv_plan_s *p) {
    int cur = -1;
    cudaError_t e = cudaGetDevice(&cur);
    if (e != cudaSuccess) {
        fc_set_error("cudaGetDevice: %s", cudaGetErrorString(e));
        return CONV_ERR_CUDA;
    }
    if (cur != p->device) {
        fc_set_error("current device %d != plan device %d", cur, p->device);
        return CONV_ERR_DEVICE_MISMATCH;
    }
    return CONV_OK;
}

static conv_status launch_result(cudaError_t e, const char *what) {
    if (e != cudaSuccess) {
        fc_set_error("%s: %s", what, cudaGetErrorString(e));
        return CONV_ERR_CUDA;
    }
    return CONV_OK;
}

static conv_status run_stage(conv_plan_s *p, const Geometry &g0, int stage, const float *in, const float *w,
                             float *out, char *ws, cudaStream_t s) {
    float *V = (float *)(ws + p->off_V);
    float *Vlo = p->gemm == CONV_GEMM_FFMA ? nullptr : (float *)(ws + p->off_Vlo);
    float *U = (float *)(ws + p->off_U);
    float *X = (float *)(ws + p->off_X);
    Geometry g = g0;
    g.umax = nullptr;
    g.vscale = nullptr;
    if (g.vf16) {
        g.umax = (unsigned int *)(ws + p->off_umax);
        g.vscale = (float *)(ws + p->off_vscale);
    }
    const int split = g.vf16 ? 2 : (Vlo != nullptr);
    if (g.nd && stage != 2) {  // N-D / non-isotropic: the generic separable transforms
        if (stage == 1 && g.vf16) {
            conv_status st = launch_result(cudaMemsetAsync(g.umax, 0, sizeof(unsigned int) * (size_t)g.B, s),
                                           "max|U_b| reset");
            if (st) return st;
        }
        static const char *names[4] = {"NK1 kernel transform (N-D)", "NK2 input transform (N-D)", "",
                                       "NK4 output transform (N-D)"};
        if (stage == 0) return launch_result(fc_launch_nd_stage(g, p->d_nd, 0, w, V, Vlo, split, s), names[0]);
        if (stage == 1) return launch_result(fc_launch_nd_stage(g, p->d_nd, 1, in, U, nullptr, 0, s), names[1]);
        if (stage == 3) return launch_result(fc_launch_nd_stage(g, p->d_nd, 3, X, out, nullptr, 0, s), names[3]);
        fc_set_error("bad stage %d", stage);
        return CONV_ERR_INVALID_ARG;
    }
    if (g.fused && (stage == 1 || stage == 3)) return CONV_OK;  // inside the fused kernel (stage 2)
    switch (stage) {
        case 0: {
            int handled = 0;
            if (!p->generic_transforms) {
                cudaError_t e = fc_launch_kernel_transform_fast(g, p->host_consts, w, V, Vlo, split, s, &handled);
                if (handled) return launch_result(e, "NK1 kernel transform");
            }
            return launch_result(fc_launch_kernel_transform(g, p->d_consts, w, V, Vlo, split, s),
                                 "NK1 kernel transform");
        }
        case 1: {
            if (g.vf16) {  // NK2 reduces max|U| for the contraction's fp16 scale
                conv_status st = launch_result(cudaMemsetAsync(g.umax, 0, sizeof(unsigned int) * (size_t)g.B, s),
                                               "max|U_b| reset");
                if (st) return st;
            }
            int handled = 0;
            if (!p->generic_transforms) {
                cudaError_t e = fc_launch_transform_fast(g, p->host_consts, in, U, 1, s, &handled);
                if (handled) return launch_result(e, "NK2 input transform");
            }
            return launch_result(fc_launch_input_transform(g, p->d_consts, in, U, s), "NK2 input transform");
        }
        case 2:
            if (g.fused)
                return launch_result(fc_launch_fused_wino23(g, in, V, Vlo, out, s), "NK2-NK4 fused F(2,3)");
            if (p->gemm == CONV_GEMM_FFMA)
                return launch_result(fc_launch_gemm_ffma(g, V, U, X, s), "NK3 FFMA contraction");
            if (g.vf16)
                return launch_result(fc_launch_gemm_tcgen05_f16(g, V, Vlo, U, X, s), "NK3 tcgen05 F16X3 contraction");
            return launch_result(fc_launch_gemm_tcgen05(g, V, Vlo, U, X, s), "NK3 tcgen05 contraction");
        case 3: {
            int handled = 0;
            if (!p->generic_transforms) {
                cudaError_t e = fc_launch_transform_fast(g, p->host_consts, X, out, 0, s, &handled);
                if (handled) return launch_result(e, "NK4 output transform");
            }
            return launch_result(fc_launch_output_transform(g, p->d_consts, X, out, s), "NK4 output transform");
        }
    }
    fc_set_error("bad stage %d", stage);
    return CONV_ERR_INVALID_ARG;
}

static conv_status check_forward_args(conv_plan_s *p, const float *in, const float *w, float *out,
                                      void *ws, size_t ws_bytes) {
    if (!p) {
        fc_set_error("NULL plan");
        return CONV_ERR_INVALID_ARG;
    }
    if (p->kind) {
        fc_set_error("a backward plan runs through conv_backward_data / conv_backward_filter only");
        return CONV_ERR_INVALID_ARG;
    }
    conv_status st = check_device(p);
    if (st) return st;
    if ((st = check_dev_ptr(p, in, "in"))) return st;
    if ((st = check_dev_ptr(p, w, "weights"))) return st;
    if ((st = check_dev_ptr(p, out, "out"))) return st;
    if (p->g.method != CONV_DIRECT) {
        if (ws_bytes < p->ws_bytes) {
            fc_set_error("workspace %zu bytes < required %zu", ws_bytes, p->ws_bytes);
            return CONV_ERR_INVALID_ARG;
        }
        if ((st = check_dev_ptr(p, ws, "workspace"))) return st;
    }
    return CONV_OK;
}

}  // extern "C"

struct conv_timer_s {
    std::vector<cudaEvent_t> ev;  // ev[i] recorded after launch i-1 (ev[0]: before the first)
    std::vector<int> stage;       // stage of the launch ending at ev[i]; -1 = start marker
    int used = 0;
};

// The whole forward pass: NK1 once (V does not depend on the batch), then
// NK2 -> NK3 -> NK4 per chunk of images so U and X stay L2-resident.
static conv_status forward_impl(conv_plan_s *p, const float *in, const float *w, float *out, char *ws,
                                cudaStream_t s, conv_timer_s *t, bool skip_nk1 = false) {
    auto mark_on = [&](int stage, cudaStream_t st_) -> conv_status {
        if (!t) return CONV_OK;
        if (t->used >= (int)t->ev.size()) {
            fc_set_error("conv_timer capacity exceeded");
            return CONV_ERR_INVALID_ARG;
        }
        t->stage[t->used] = stage;
        return launch_result(cudaEventRecord(t->ev[t->used++], st_), "cudaEventRecord");
    };
    auto mark = [&](int stage) { return mark_on(stage, s); };
    const Geometry &g = p->g;
    conv_status st;
    if (g.method == CONV_DIRECT) {
        if ((st = mark(-1))) return st;
        st = launch_result(g.nd ? fc_launch_nd_direct(g, in, w, out, s) : fc_launch_direct(g, in, w, out, s),
                           "NK5 direct");
        return st ? st : mark(2);
    }
    // NK1 (V from the weights) and NK2 (U from the input) are independent: with overlap on,
    // NK1 runs on the plan's auxiliary stream concurrently with NK2, and the first NK3 waits
    // for both (fork / join events; captured as parallel branches inside CUDA graphs)
    cudaEvent_t join = nullptr;
    if (!skip_nk1) {
        if (p->overlap_nk1) {
            const unsigned k = __atomic_fetch_add(&p->evc, 1u, __ATOMIC_RELAXED) % FC_EVPAIRS;
            join = p->join_ev[k];
            if ((st = launch_result(cudaEventRecord(p->fork_ev[k], s), "fork")) ||
                (st = launch_result(cudaStreamWaitEvent(p->aux, p->fork_ev[k], 0), "fork wait")) ||
                (st = mark_on(-1, p->aux)) || (st = run_stage(p, g, 0, in, w, out, ws, p->aux)) ||
                (st = mark_on(0, p->aux)) || (st = launch_result(cudaEventRecord(join, p->aux), "join")))
                return st;
        } else if ((st = mark(-1)) || (st = run_stage(p, g, 0, in, w, out, ws, s)) || (st = mark(0))) {
            return st;
        }
    }
    if ((st = mark(-1))) return st;
    for (int b0 = 0; b0 < g.B; b0 += p->chunk) {
        const Geometry gc = fc_chunk_geometry(g, g.B - b0 < p->chunk ? g.B - b0 : p->chunk);
        const float *in_c = in + (size_t)b0 * g.C * (size_t)g.vin;
        float *out_c = out + (size_t)b0 * g.Cout * (size_t)g.vout;
        for (int k = 1; k < 4; ++k) {
            if (k == 2 && join) {
                if ((st = launch_result(cudaStreamWaitEvent(s, join, 0), "join wait"))) return st;
                join = nullptr;
            }
            if ((st = run_stage(p, gc, k, in_c, w, out_c, ws, s)) || (st = mark(k))) return st;
        }
    }
    return CONV_OK;
}

extern "C" {

conv_status conv_forward(conv_plan_t p, const float *in, const float *w, float *out, void *ws,
                         size_t ws_bytes, void *stream) {
    conv_status st = check_forward_args(p, in, w, out, ws, ws_bytes);
    if (st) return st;
    return forward_impl(p, in, w, out, (char *)ws, (cudaStream_t)stream, nullptr);
}

conv_status conv_transform_weights(conv_plan_t p, const float *w, void *ws, size_t ws_bytes, void *stream) {
    if (!p) {
        fc_set_error("NULL plan");
        return CONV_ERR_INVALID_ARG;
    }
    if (p->kind) {
        fc_set_error("a backward plan runs through conv_backward_data / conv_backward_filter only");
        return CONV_ERR_INVALID_ARG;
    }
    if (p->g.method == CONV_DIRECT) {
        fc_set_error("direct plans have no kernel transform");
        return CONV_ERR_UNSUPPORTED;
    }
    conv_status st = check_device(p);
    if (st) return st;
    if ((st = check_dev_ptr(p, w, "weights"))) return st;
    if (ws_bytes < p->ws_bytes) {
        fc_set_error("workspace %zu bytes < required %zu", ws_bytes, p->ws_bytes);
        return CONV_ERR_INVALID_ARG;
    }
    if ((st = check_dev_ptr(p, ws, "workspace"))) return st;
    return run_stage(p, p->g, 0, nullptr, w, nullptr, (char *)ws, (cudaStream_t)stream);
}

conv_status conv_forward_cached(conv_plan_t p, const float *in, float *out, void *ws, size_t ws_bytes,
                                void *stream) {
    if (!p) {
        fc_set_error("NULL plan");
        return CONV_ERR_INVALID_ARG;
    }
    if (p->kind) {
        fc_set_error("a backward plan runs through conv_backward_data / conv_backward_filter only");
        return CONV_ERR_INVALID_ARG;
    }
    if (p->g.method == CONV_DIRECT) {
        fc_set_error("direct plans have no transformed weights");
        return CONV_ERR_UNSUPPORTED;
    }
    conv_status st = check_device(p);
    if (st) return st;
    if ((st = check_dev_ptr(p, in, "in"))) return st;
    if ((st = check_dev_ptr(p, out, "out"))) return st;
    if (ws_bytes < p->ws_bytes) {
        fc_set_error("workspace %zu bytes < required %zu", ws_bytes, p->ws_bytes);
        return CONV_ERR_INVALID_ARG;
    }
    if ((st = check_dev_ptr(p, ws, "workspace"))) return st;
    return forward_impl(p, in, nullptr, out, (char *)ws, (cudaStream_t)stream, nullptr, true);
}

conv_status conv_run_stage(conv_plan_t p, int stage, const float *in, const float *w, float *out,
                           void *ws, size_t ws_bytes, void *stream) {
    if (!p) {
        fc_set_error("NULL plan");
        return CONV_ERR_INVALID_ARG;
    }
    if (p->kind) {
        fc_set_error("a backward plan runs through conv_backward_data / conv_backward_filter only");
        return CONV_ERR_INVALID_ARG;
    }
    if (p->g.method == CONV_DIRECT) {
        fc_set_error("direct plans have no stages");
        return CONV_ERR_UNSUPPORTED;
    }
    conv_status st = check_device(p);
    if (st) return st;
    if (ws_bytes < p->ws_bytes) {
        fc_set_error("workspace %zu bytes < required %zu", ws_bytes, p->ws_bytes);
        return CONV_ERR_INVALID_ARG;
    }
    if ((st = check_dev_ptr(p, ws, "workspace"))) return st;
    if (stage == 0 && (st = check_dev_ptr(p, w, "weights"))) return st;
    if (stage == 1 && (st = check_dev_ptr(p, in, "in"))) return st;
    if (stage == 3 && (st = check_dev_ptr(p, out, "out"))) return st;
    const Geometry g0 = stage == 0 ? p->g : fc_chunk_geometry(p->g, p->chunk);
    return run_stage(p, g0, stage, in, w, out, (char *)ws, (cudaStream_t)stream);
}

conv_status conv_timer_create(conv_timer_t *t, int max_launches) {
    if (!t || max_launches < 1) {
        fc_set_error("bad timer arguments");
        return CONV_ERR_INVALID_ARG;
    }
    conv_timer_s *tm = new (std::nothrow) conv_timer_s();
    if (!tm) return CONV_ERR_OUT_OF_MEMORY;
    tm->ev.resize((size_t)max_launches + 64);
    tm->stage.assign(tm->ev.size(), -1);
    for (size_t i = 0; i < tm->ev.size(); ++i) {
        if (cudaEventCreate(&tm->ev[i]) != cudaSuccess) {
            for (size_t j = 0; j < i; ++j) cudaEventDestroy(tm->ev[j]);
            delete tm;
            return launch_result(cudaGetLastError(), "cudaEventCreate");
        }
    }
    *t = tm;
    return CONV_OK;
}

void conv_timer_reset(conv_timer_t t) {
    if (t) t->used = 0;
}

void conv_timer_destroy(conv_timer_t t) {
    if (!t) return;
    for (cudaEvent_t e : t->ev) cudaEventDestroy(e);
    delete t;
}

conv_status conv_forward_timed(conv_plan_t p, const float *in, const float *w, float *out, void *ws,
                               size_t ws_bytes, void *stream, conv_timer_t t) {
    if (!t) {
        fc_set_error("NULL timer");
        return CONV_ERR_INVALID_ARG;
    }
    conv_status st = check_forward_args(p, in, w, out, ws, ws_bytes);
    if (st) return st;
    return forward_impl(p, in, w, out, (char *)ws, (cudaStream_t)stream, t);
}

conv_status conv_timer_read(conv_timer_t t, float stage_ms[4], int *launches) {
    if (!t || !stage_ms) {
        fc_set_error("NULL argument");
        return CONV_ERR_INVALID_ARG;
    }
    for (int k = 0; k < 4; ++k) stage_ms[k] = 0.f;
    int n = 0;
    if (t->used > 0) {
        cudaError_t e = cudaEventSynchronize(t->ev[t->used - 1]);
        if (e != cudaSuccess) return launch_result(e, "cudaEventSynchronize");
    }
    for (int i = 1; i < t->used; ++i) {
        if (t->stage[i] < 0) continue;  // start marker of the next forward call
        float ms = 0.f;
        cudaError_t e = cudaEventElapsedTime(&ms, t->ev[i - 1], t->ev[i]);
        if (e != cudaSuccess) return launch_result(e, "cudaEventElapsedTime");
        stage_ms[t->stage[i]] += ms;
        ++n;
    }
    if (launches) *launches = n;
    return CONV_OK;
}

conv_status conv_forward_profiled(conv_plan_t p, const float *in, const float *w, float *out,
                                  void *ws, size_t ws_bytes, void *stream, float stage_ms[4]) {
    conv_status st = check_forward_args(p, in, w, out, ws, ws_bytes);
    if (st) return st;
    if (!stage_ms) {
        fc_set_error("NULL stage_ms");
        return CONV_ERR_INVALID_ARG;
    }
    conv_timer_t t = nullptr;
    if ((st = conv_timer_create(&t, conv_forward_launch_count(p)))) return st;
    st = forward_impl(p, in, w, out, (char *)ws, (cudaStream_t)stream, t);
    if (!st) st = conv_timer_read(t, stage_ms, nullptr);
    conv_timer_destroy(t);
    return st;
}

conv_status conv_forward_host(conv_plan_t p, const float *h_in, const float *h_w, float *h_out,
                              float *d_in, float *d_w, float *d_out, void *ws, size_t ws_bytes,
                              void *stream) {
    if (!p || !h_in || !h_w || !h_out) {
        fc_set_error("NULL argument");
        return CONV_ERR_INVALID_ARG;
    }
    conv_status st = check_forward_args(p, d_in, d_w, d_out, ws, ws_bytes);
    if (st) return st;
    const Geometry &g = p->g;
    cudaStream_t s = (cudaStream_t)stream;
    const size_t img_in = (size_t)g.C * (size_t)g.vin, img_out = (size_t)g.Cout * (size_t)g.vout;
    const size_t nw = (size_t)g.Cout * g.C * (size_t)g.kvol * 4;
    cudaError_t e = cudaMemcpyAsync(d_w, h_w, nw, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return launch_result(e, "H2D copy (weights)");
    if (g.method != CONV_DIRECT && p->e2e_chunks > 1 && !p->h2d) {  // first host call: copy streams
        static std::mutex mu;
        std::lock_guard<std::mutex> lock(mu);
        if (!p->h2d) {
            cudaStream_t a = nullptr, b = nullptr;
            if (cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking) == cudaSuccess &&
                cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking) == cudaSuccess) {
                p->d2h = b;
                __atomic_store_n(&p->h2d, a, __ATOMIC_RELEASE);
            } else {  // falls back to the serial host path
                cudaGetLastError();
                if (a) cudaStreamDestroy(a);
            }
        }
    }
    if (g.method == CONV_DIRECT || !p->h2d || !p->d2h) {
        e = cudaMemcpyAsync(d_in, h_in, img_in * g.B * 4, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return launch_result(e, "H2D copy");
        if ((st = forward_impl(p, d_in, d_w, d_out, (char *)ws, s, nullptr))) return st;
        return launch_result(cudaMemcpyAsync(h_out, d_out, img_out * g.B * 4, cudaMemcpyDeviceToHost, s),
                             "D2H copy");
    }
    // Pipelined over image chunks: the H2D of chunk i+1 (copy stream), the kernels of
    // chunk i (caller's stream) and the D2H of chunk i-1 (second copy stream) overlap;
    // PCIe runs both directions at once.  The plan's own chunk (<= this one) sizes U / X.
    const int nck = p->e2e_chunks < g.B ? p->e2e_chunks : g.B;
    // chunk boundaries: half-size first and last chunks (the first H2D and the last D2H are the
    // pipeline's exposed ends), the rest split evenly
    std::vector<int> bnd(1, 0);
    {
        const int edge = nck >= 3 ? std::max(1, g.B / (2 * nck)) : 0;
        const int mid = g.B - 2 * edge, nm = nck >= 3 ? nck - 2 : nck;
        if (edge) bnd.push_back(edge);
        for (int k = 1; k <= nm; ++k) bnd.push_back(edge + (int)((long long)mid * k / nm));
        if (edge) bnd.push_back(g.B);
    }
    std::vector<cudaEvent_t> evs;
    auto mk = [&]() -> cudaEvent_t {
        cudaEvent_t ev = nullptr;
        if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess) evs.push_back(ev);
        return ev;
    };
    cudaEvent_t start = mk();
    e = cudaEventRecord(start, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->h2d, start, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->d2h, start, 0);
    if (e == cudaSuccess && (st = run_stage(p, g, 0, nullptr, d_w, nullptr, (char *)ws, s))) {
        for (cudaEvent_t ev : evs) cudaEventDestroy(ev);
        return st;
    }
    for (size_t ci = 0; ci + 1 < bnd.size() && e == cudaSuccess && !st; ++ci) {
        const int b0 = bnd[ci], nb = bnd[ci + 1] - bnd[ci];
        if (nb <= 0) continue;
        cudaEvent_t in_ready = mk(), out_ready = mk();
        if (!in_ready || !out_ready) {
            e = cudaErrorMemoryAllocation;
            break;
        }
        e = cudaMemcpyAsync(d_in + (size_t)b0 * img_in, h_in + (size_t)b0 * img_in, (size_t)nb * img_in * 4,
                            cudaMemcpyHostToDevice, p->h2d);
        if (e == cudaSuccess) e = cudaEventRecord(in_ready, p->h2d);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, in_ready, 0);
        if (e != cudaSuccess) break;
        for (int c0 = 0; c0 < nb && !st; c0 += p->chunk) {
            const int bc = nb - c0 < p->chunk ? nb - c0 : p->chunk;
            const Geometry gc = fc_chunk_geometry(g, bc);
            const float *in_c = d_in + (size_t)(b0 + c0) * img_in;
            float *out_c = d_out + (size_t)(b0 + c0) * img_out;
            for (int k = 1; k < 4 && !st; ++k) st = run_stage(p, gc, k, in_c, d_w, out_c, (char *)ws, s);
        }
        if (st) break;
        e = cudaEventRecord(out_ready, s);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(p->d2h, out_ready, 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(h_out + (size_t)b0 * img_out, d_out + (size_t)b0 * img_out, (size_t)nb * img_out * 4,
                                cudaMemcpyDeviceToHost, p->d2h);
    }
    cudaEvent_t done = mk();
    if (e == cudaSuccess && done) e = cudaEventRecord(done, p->d2h);
    if (e == cudaSuccess && done) e = cudaStreamWaitEvent(s, done, 0);  // caller's stream sees the D2H
    for (cudaEvent_t ev : evs) cudaEventDestroy(ev);                     // released once completed
    if (st) return st;
    return launch_result(e, "pipelined host forward");
}


// -- CUDA graphs -----------------------------------------------------------------
struct conv_graph_s {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int device = 0;
};

void conv_graph_destroy(conv_graph_t gr) {
    if (!gr) return;
    if (gr->exec) cudaGraphExecDestroy(gr->exec);
    if (gr->graph) cudaGraphDestroy(gr->graph);
    delete gr;
}

conv_status conv_graph_create(conv_plan_t p, const float *in, const float *w, float *out, void *ws,
                              size_t ws_bytes, int steps, int cached, conv_graph_t *out_graph) {
    if (!out_graph || steps < 1) {
        fc_set_error("NULL graph pointer or steps < 1");
        return CONV_ERR_INVALID_ARG;
    }
    *out_graph = nullptr;
    conv_status st;
    if (p && p->kind) {
        fc_set_error("a backward plan runs through conv_backward_data / conv_backward_filter only");
        return CONV_ERR_INVALID_ARG;
    }
    if (cached) {
        if (!p || p->g.method == CONV_DIRECT) {
            fc_set_error("cached graphs need a fast-method plan");
            return p ? CONV_ERR_UNSUPPORTED : CONV_ERR_INVALID_ARG;
        }
        if ((st = check_device(p))) return st;
        if ((st = check_dev_ptr(p, in, "in")) || (st = check_dev_ptr(p, out, "out")) ||
            (st = check_dev_ptr(p, ws, "workspace")))
            return st;
        if (ws_bytes < p->ws_bytes) {
            fc_set_error("workspace %zu bytes < required %zu", ws_bytes, p->ws_bytes);
            return CONV_ERR_INVALID_ARG;
        }
    } else if ((st = check_forward_args(p, in, w, out, ws, ws_bytes))) {
        return st;
    }
    conv_graph_s *gr = new (std::nothrow) conv_graph_s();
    if (!gr) return CONV_ERR_OUT_OF_MEMORY;
    gr->device = p->device;
    cudaStream_t cs = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
        if (cs) cudaStreamDestroy(cs);
        delete gr;
        return launch_result(e, "graph capture begin");
    }
    for (int i = 0; i < steps && !st; ++i)
        st = forward_impl(p, in, w, out, (char *)ws, cs, nullptr, cached != 0);
    cudaGraph_t graph = nullptr;
    e = cudaStreamEndCapture(cs, &graph);
    cudaStreamDestroy(cs);
    if (st || e != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        delete gr;
        return st ? st : launch_result(e, "graph capture end");
    }
    gr->graph = graph;
    e = cudaGraphInstantiate(&gr->exec, graph, 0);
    if (e != cudaSuccess) {
        conv_graph_destroy(gr);
        return launch_result(e, "graph instantiate");
    }
    *out_graph = gr;
    return CONV_OK;
}

conv_status conv_graph_launch(conv_graph_t gr, void *stream) {
    if (!gr || !gr->exec) {
        fc_set_error("NULL graph");
        return CONV_ERR_INVALID_ARG;
    }
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != gr->device) {
        fc_set_error("current device %d != graph device %d", cur, gr->device);
        return CONV_ERR_DEVICE_MISMATCH;
    }
    return launch_result(cudaGraphLaunch(gr->exec, (cudaStream_t)stream), "graph launch");
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Element-sharded execution (the contraction's E independent
// products): rank j of g owns the transformed elements e in [e0_j, e1_j)
// (parallel.shard_range over E) for EVERY image, and its own images b in [lo_j, hi_j) for
// the transforms:
//   a) NK1 for its elements only (V_j: E_j / E of V -- no replicated kernel transform),
//      NK2 for its images (U_local, per-image max|U_b|), U packed per destination peer;
//   -- caller: all-to-all of U (peer-major chunks) and all-gather of the per-image max|U_b|
//   b) NK3 for its elements over all B N columns (the received chunks are one U operand
//      [sum_k NB_k][Z_j][K][128]; F16X3 scales per column from the gathered maxima),
//      X_j packed per destination peer (its images' columns);
//   -- caller: all-to-all of X
//   c) X chunks placed into X_local [Xz][Xm][BN_pad], NK4 for its images.
// Every per-column computation is the one the batch-sharded / single-GPU plan performs
// (same V entries, same K order, same per-image scale), so results are bit-identical to
// conv_forward on the whole batch.
// ---------------------------------------------------------------------------
struct conv_eshard_s {
    int world, rank;
    std::vector<int> blo, bcnt;           // images per rank (prefix / count)
    std::vector<int> elo, ecnt;           // elements per rank
    std::vector<long long> bnpad;         // per rank: its images' B_k N columns padded to 128
    long long bn_tot;                     // sum of bnpad
    conv_plan_s *lp;                      // local plan: this rank's images, all E (NK2 / NK4)
    conv_plan_s lpx;                      // the same plan with this workspace's U / X / max offsets
    char *d_seg;                          // device table: per-peer column offset, B_k N, first image
    char *d_peer;                         // device: up to 8 peer X tensor maps (128 B each) + first columns
    Geometry gv;                          // NK1 over [e0, e1) (generic kernel, full-E indices)
    Geometry gj;                          // NK3 on E_j elements, bn_tot columns (N = 1)
    int pu, px;                           // plane groups of U / X (3 for Gauss three-plane, else 1)
    size_t off_V, off_Vlo, off_vscale, off_umaxc, off_Xj, off_U, off_X, off_umaxl, ws_bytes;
    std::vector<size_t> u_send, u_recv, x_send, x_recv;
};

static int split_lo(int n, int k, int w) { return k * (n / w) + (k < n % w ? k : n % w); }

// byte offset of sender j's segment in receiver k's U / X receive buffer (segments in rank order)
static size_t eshard_u_recv_off(const conv_eshard_s *e, int k, int j) {
    const Geometry &g = e->lp->g;
    size_t off = 0;
    for (int i = 0; i < j; ++i) off += (size_t)(e->bnpad[i] / FC_TB) * e->pu * e->ecnt[k] * g.K * FC_TB * 4;
    return off;
}
static size_t eshard_x_recv_off(const conv_eshard_s *e, int k, int j) {
    const Geometry &g = e->lp->g;
    size_t off = 0;
    for (int i = 0; i < j; ++i) off += (size_t)e->px * e->ecnt[i] * g.Xm * e->bnpad[k] * 4;
    return off;
}

extern "C" {

conv_status conv_eshard_create(conv_eshard_t *out, int world, int rank, const int *batch, int C, int Cout, int H,
                               int W, int r, conv_method method, int m, const conv_plan_options *opts_in) {
    if (!out || !batch || world < 1 || rank < 0 || rank >= world || method == CONV_DIRECT) {
        fc_set_error("conv_eshard_create: bad rank / world / batch or the direct method");
        return CONV_ERR_INVALID_ARG;
    }
    conv_plan_options opts;
    if (opts_in) {
        conv_status st = check_options(opts_in);
        if (st) return st;
        opts = *opts_in;
    } else {
        conv_plan_options_init(&opts);
    }
    opts.chunk_images = 0;
    if (opts.fused) {  // the exchange needs U and X in memory
        fc_set_error("conv_eshard_create: fused plans keep U and X on chip; element sharding needs them");
        return CONV_ERR_UNSUPPORTED;
    }
    int Btot = 0;
    for (int k = 0; k < world; ++k) {
        if (batch[k] < 1) {
            fc_set_error("conv_eshard_create: every rank needs >= 1 image (rank %d has %d)", k, batch[k]);
            return CONV_ERR_INVALID_ARG;
        }
        Btot += batch[k];
    }
    conv_eshard_s *e = new (std::nothrow) conv_eshard_s();
    if (!e) return CONV_ERR_OUT_OF_MEMORY;
    e->world = world;
    e->rank = rank;
    conv_plan_t lp = nullptr;
    conv_status st = plan_create(&lp, 0, batch[rank], C, Cout, H, W, r, method, m, nullptr, nullptr, nullptr, &opts);
    if (st) {
        delete e;
        return st;
    }
    e->lp = lp;
    const Geometry &g = lp->g;
    if (g.E < world) {
        conv_destroy(lp);
        delete e;
        fc_set_error("conv_eshard_create: %d elements cannot be split over %d ranks", g.E, world);
        return CONV_ERR_UNSUPPORTED;
    }
    int acc = 0;
    e->bn_tot = 0;
    for (int k = 0; k < world; ++k) {
        e->blo.push_back(acc);
        e->bcnt.push_back(batch[k]);
        acc += batch[k];
        const long long bn = (long long)batch[k] * g.N;
        e->bnpad.push_back((bn + FC_TB - 1) / FC_TB * FC_TB);
        e->bn_tot += e->bnpad.back();
        const int lo = split_lo(g.E, k, world), hi = split_lo(g.E, k + 1, world);
        e->elo.push_back(lo);
        e->ecnt.push_back(hi - lo);
    }
    e->pu = g.method == CONV_GAUSS_FFT ? 3 : 1;
    e->px = (g.method == CONV_GAUSS_FFT && !g.gc) ? 3 : 1;
    const int Ej = e->ecnt[rank];
    // NK1 geometry: the generic kernel writes e in [e0, e1) relative to e0
    e->gv = g;
    e->gv.e_lo = e->elo[rank];
    e->gv.e_hi = e->elo[rank] + Ej;
    // NK3 geometry: E_j elements, every rank's (padded) columns, one "tile per image" so the
    // F16X3 scale of column n is the per-column maximum built from the gathered per-image ones
    Geometry gj = g;
    gj.E = Ej;
    gj.e_lo = 0;
    gj.e_hi = Ej;
    gj.Z = e->pu * Ej;
    gj.Xz = g.gc ? Ej : gj.Z;
    gj.B = (int)e->bn_tot;
    gj.N = 1;
    gj.divN = fc_fastdiv(1);
    gj.BN = e->bn_tot;
    gj.BN_pad = e->bn_tot;
    e->gj = gj;
    // workspace: V_j (hi, lo, scales), per-column maxima, X_j, then the local U / X / max|U_b|
    const size_t vb = fc_v_bytes(gj);
    size_t off = 0;
    e->off_V = off;
    off += align256(vb);
    e->off_Vlo = lp->gemm == CONV_GEMM_FFMA ? 0 : off;
    if (lp->gemm != CONV_GEMM_FFMA) off += align256(vb);
    e->off_vscale = off;
    off += align256((size_t)2 * Cout * 4);
    e->off_umaxc = off;
    off += align256((size_t)e->bn_tot * 4);
    e->off_Xj = off;
    off += align256((size_t)gj.Xz * gj.Xm * e->bn_tot * 4);
    e->off_U = off;
    off += align256(lp->info.bytes_U);
    e->off_X = off;
    off += align256(lp->info.bytes_X);
    e->off_umaxl = off;
    off += align256((size_t)batch[rank] * 4);
    e->ws_bytes = off;
    e->lpx = *lp;
    e->lpx.off_U = e->off_U;
    e->lpx.off_X = e->off_X;
    e->lpx.off_umax = e->off_umaxl;
    {  // per-peer segments of the contraction's columns (for the per-column F16X3 maxima)
        std::vector<char> host((size_t)world * 20);
        long long c0 = 0;
        for (int k = 0; k < world; ++k) {
            const long long bn = (long long)batch[k] * g.N;
            memcpy(host.data() + (size_t)k * 8, &c0, 8);
            memcpy(host.data() + (size_t)world * 8 + (size_t)k * 8, &bn, 8);
            memcpy(host.data() + (size_t)world * 16 + (size_t)k * 4, &e->blo[k], 4);
            c0 += e->bnpad[k];
        }
        cudaError_t ce = cudaMalloc(&e->d_seg, host.size());
        if (ce == cudaSuccess) ce = cudaMemcpy(e->d_seg, host.data(), host.size(), cudaMemcpyHostToDevice);
        if (ce != cudaSuccess) {
            if (e->d_seg) cudaFree(e->d_seg);
            conv_destroy(lp);
            delete e;
            fc_set_error("e-shard segment table: %s", cudaGetErrorString(ce));
            return CONV_ERR_CUDA;
        }
    }
    // tensor maps of the peers' X receive buffers (contraction epilogue -> peers), world <= 8
    if (world <= 8 && cudaMalloc(&e->d_peer, 8 * 128 + 8 * 8) != cudaSuccess) {
        cudaGetLastError();
        e->d_peer = nullptr;  // the peer exchange then packs X with copies
    }
    // per-peer message sizes (bytes)
    const long long NBme = e->bnpad[rank] / FC_TB;
    for (int k = 0; k < world; ++k) {
        e->u_send.push_back((size_t)NBme * e->pu * e->ecnt[k] * g.K * FC_TB * 4);
        e->u_recv.push_back((size_t)(e->bnpad[k] / FC_TB) * e->pu * Ej * g.K * FC_TB * 4);
        e->x_send.push_back((size_t)e->px * Ej * g.Xm * e->bnpad[k] * 4);
        e->x_recv.push_back((size_t)e->px * e->ecnt[k] * g.Xm * e->bnpad[rank] * 4);
    }
    *out = e;
    return CONV_OK;
}

void conv_eshard_destroy(conv_eshard_t e) {
    if (!e) return;
    if (e->d_seg) cudaFree(e->d_seg);
    if (e->d_peer) cudaFree(e->d_peer);
    conv_destroy(e->lp);
    delete e;
}

conv_status conv_eshard_sizes(conv_eshard_t e, size_t *workspace_bytes, size_t *u_send, size_t *u_recv,
                              size_t *x_send, size_t *x_recv) {
    if (!e) {
        fc_set_error("NULL e-shard plan");
        return CONV_ERR_INVALID_ARG;
    }
    if (workspace_bytes) *workspace_bytes = e->ws_bytes;
    for (int k = 0; k < e->world; ++k) {
        if (u_send) u_send[k] = e->u_send[k];
        if (u_recv) u_recv[k] = e->u_recv[k];
        if (x_send) x_send[k] = e->x_send[k];
        if (x_recv) x_recv[k] = e->x_recv[k];
    }
    return CONV_OK;
}

conv_status conv_eshard_get_info(conv_eshard_t e, conv_plan_info *local, int *e_lo, int *e_count) {
    if (!e) {
        fc_set_error("NULL e-shard plan");
        return CONV_ERR_INVALID_ARG;
    }
    if (local) *local = e->lp->info;
    if (e_lo) *e_lo = e->elo[e->rank];
    if (e_count) *e_count = e->ecnt[e->rank];
    return CONV_OK;
}

static conv_status eshard_check(conv_eshard_s *e, void *ws, size_t ws_bytes) {
    if (!e) {
        fc_set_error("NULL e-shard plan");
        return CONV_ERR_INVALID_ARG;
    }
    conv_status st = check_device(e->lp);
    if (st) return st;
    if (ws_bytes < e->ws_bytes) {
        fc_set_error("workspace %zu bytes < required %zu", ws_bytes, e->ws_bytes);
        return CONV_ERR_INVALID_ARG;
    }
    return check_dev_ptr(e->lp, ws, "workspace");
}

static conv_status eshard_forward_a_impl(conv_eshard_t e, const float *in, const float *w, void *u_send,
                                         void *const *u_recv_peer, float *umax_out, void *ws, size_t ws_bytes,
                                         void *stream) {
    conv_status st = eshard_check(e, ws, ws_bytes);
    if (st) return st;
    if ((st = check_dev_ptr(e->lp, in, "in")) || (st = check_dev_ptr(e->lp, w, "weights"))) return st;
    if (u_recv_peer) {
        for (int k = 0; k < e->world; ++k)
            if (!u_recv_peer[k]) {
                fc_set_error("u_recv_peer[%d] is NULL", k);
                return CONV_ERR_INVALID_ARG;
            }
    } else if ((st = check_dev_ptr(e->lp, u_send, "u_send"))) {
        return st;
    }
    cudaStream_t s = (cudaStream_t)stream;
    char *b = (char *)ws;
    conv_plan_s *lp = e->lp;
    // NK1 for this rank's elements (generic kernel with the element range)
    Geometry gv = e->gv;
    gv.vscale = (float *)(b + e->off_vscale);
    gv.umax = nullptr;
    const int split = gv.vf16 ? 2 : (e->off_Vlo ? 1 : 0);
    {  // the same NK1 kernel the whole-batch plan runs (codelet or generic), on the element range
        float *Vj = (float *)(b + e->off_V), *Vjlo = e->off_Vlo ? (float *)(b + e->off_Vlo) : nullptr;
        int handled = 0;
        cudaError_t ce = cudaSuccess;
        if (!lp->generic_transforms)
            ce = fc_launch_kernel_transform_fast(gv, lp->host_consts, w, Vj, Vjlo, split, s, &handled);
        if (!handled) ce = fc_launch_kernel_transform(gv, lp->d_consts, w, Vj, Vjlo, split, s);
        if ((st = launch_result(ce, "NK1 kernel transform (element shard)"))) return st;
    }
    // NK2 for this rank's images into U_local (per-image maxima into the local slot)
    if ((st = run_stage(&e->lpx, lp->g, 1, in, nullptr, nullptr, b, s))) return st;
    if (umax_out) {
        if ((st = check_dev_ptr(lp, umax_out, "umax_out"))) return st;
        if (lp->g.vf16)
            st = launch_result(cudaMemcpyAsync(umax_out, b + e->off_umaxl, (size_t)lp->g.B * 4,
                                               cudaMemcpyDeviceToDevice, s), "max|U_b| copy");
        else
            st = launch_result(cudaMemsetAsync(umax_out, 0, (size_t)lp->g.B * 4, s), "max|U_b| clear");
        if (st) return st;
    }
    // pack U_local [NB][Z][K][128] -> peer j: [NB][pu][E_j][K][128], into the send buffer
    // (peer-major) or straight into peer j's receive buffer at this rank's segment
    const Geometry &g = lp->g;
    const size_t row = (size_t)g.K * FC_TB * 4;  // one (z) slab of a 128-tile block
    const long long NB = e->bnpad[e->rank] / FC_TB;
    char *dst = (char *)u_send;
    for (int j = 0; j < e->world; ++j) {
        const int Ej = e->ecnt[j];
        if (u_recv_peer) dst = (char *)u_recv_peer[j] + eshard_u_recv_off(e, j, e->rank);
        for (int p = 0; p < e->pu; ++p) {
            const char *src = b + e->off_U + (size_t)(p * g.E + e->elo[j]) * row;
            st = launch_result(cudaMemcpy2DAsync(dst + (size_t)p * Ej * row, (size_t)e->pu * Ej * row, src,
                                                 (size_t)g.Z * row, (size_t)Ej * row, (size_t)NB,
                                                 cudaMemcpyDeviceToDevice, s),
                               "U pack");
            if (st) return st;
        }
        dst += e->u_send[j];
    }
    return CONV_OK;
}

conv_status conv_eshard_forward_a(conv_eshard_t e, const float *in, const float *w, void *u_send, float *umax_out,
                                  void *ws, size_t ws_bytes, void *stream) {
    return eshard_forward_a_impl(e, in, w, u_send, nullptr, umax_out, ws, ws_bytes, stream);
}

conv_status conv_eshard_forward_a_peer(conv_eshard_t e, const float *in, const float *w, void *const *u_recv_peer,
                                       float *umax_out, void *ws, size_t ws_bytes, void *stream) {
    if (!u_recv_peer) {
        fc_set_error("NULL u_recv_peer array");
        return CONV_ERR_INVALID_ARG;
    }
    return eshard_forward_a_impl(e, in, w, nullptr, u_recv_peer, umax_out, ws, ws_bytes, stream);
}

}  // extern "C"

namespace {
// per-column F16X3 maxima of the element shard's contraction: column n of peer k's segment
// (offset off_k) is tile n - off_k of peer k's images, image lo_k + (n - off_k) / N
__global__ void eshard_col_umax(unsigned int *col, const unsigned int *img, const long long *seg_off,
                                const int *seg_lo, const long long *seg_bn, int world, int N, long long total) {
    for (long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x; n < total;
         n += (long long)gridDim.x * blockDim.x) {
        int k = 0;
        while (k + 1 < world && n >= seg_off[k + 1]) ++k;
        const long long t = n - seg_off[k];
        col[n] = t < seg_bn[k] ? img[seg_lo[k] + (int)(t / N)] : 0u;
    }
}
}  // namespace

extern "C" {

static conv_status eshard_forward_b_impl(conv_eshard_t e, const void *u_recv, const float *umax_all, void *x_send,
                                         void *const *x_recv_peer, void *ws, size_t ws_bytes, void *stream) {
    conv_status st = eshard_check(e, ws, ws_bytes);
    if (st) return st;
    if ((st = check_dev_ptr(e->lp, u_recv, "u_recv"))) return st;
    if (x_recv_peer) {
        for (int k = 0; k < e->world; ++k)
            if (!x_recv_peer[k]) {
                fc_set_error("x_recv_peer[%d] is NULL", k);
                return CONV_ERR_INVALID_ARG;
            }
    } else if ((st = check_dev_ptr(e->lp, x_send, "x_send"))) {
        return st;
    }
    cudaStream_t s = (cudaStream_t)stream;
    char *b = (char *)ws;
    conv_plan_s *lp = e->lp;
    Geometry gj = e->gj;
    gj.vscale = (float *)(b + e->off_vscale);
    gj.umax = nullptr;
    float *V = (float *)(b + e->off_V);
    float *Vlo = e->off_Vlo ? (float *)(b + e->off_Vlo) : nullptr;
    float *Xj = (float *)(b + e->off_Xj);
    const float *U = (const float *)u_recv;
    if (gj.vf16) {
        if (!umax_all || (st = check_dev_ptr(lp, umax_all, "umax_all"))) {
            if (!st) fc_set_error("F16X3 element shards need the gathered per-image max|U_b|");
            return st ? st : CONV_ERR_INVALID_ARG;
        }
        const int w = e->world;
        const char *dtab = e->d_seg;
        unsigned int *col = (unsigned int *)(b + e->off_umaxc);
        const long long total = e->bn_tot;
        eshard_col_umax<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(
            col, (const unsigned int *)umax_all, (const long long *)dtab, (const int *)(dtab + (size_t)w * 16),
            (const long long *)(dtab + (size_t)w * 8), w, lp->g.N, total);
        if ((st = launch_result(cudaGetLastError(), "per-column maxima"))) return st;
        gj.umax = col;
    }
    // peer exchange with a tcgen05 contraction (not the Gauss combine): the epilogue stores each
    // X box straight into its owner's receive buffer through per-peer tensor maps
    const bool fuse_x = x_recv_peer && e->d_peer && lp->gemm != CONV_GEMM_FFMA && !gj.gc;
    if (fuse_x) {
        alignas(64) unsigned char maps[8][128];
        long long cols[8];
        long long c0 = 0;
        for (int k = 0; k < e->world; ++k) {
            const unsigned long long bp = (unsigned long long)e->bnpad[k];
            const unsigned long long dims[3] = {bp, (unsigned long long)gj.Xm, (unsigned long long)gj.Xz};
            const unsigned long long strides[2] = {bp * 4ull, (unsigned long long)gj.Xm * bp * 4ull};
            const unsigned int box[3] = {32, 32, 1};
            if (!fc_tma_encode_f32(maps[k], (char *)x_recv_peer[k] + eshard_x_recv_off(e, k, e->rank), 3, dims,
                                   strides, box, 128)) {
                fc_set_error("tensor map of peer %d's X receive buffer", k);
                return CONV_ERR_CUDA;
            }
            cols[k] = c0;
            c0 += e->bnpad[k];
        }
        if ((st = launch_result(cudaMemcpyAsync(e->d_peer, maps, (size_t)e->world * 128, cudaMemcpyHostToDevice, s),
                                "peer tensor maps")) ||
            (st = launch_result(cudaMemcpyAsync(e->d_peer + 8 * 128, cols, (size_t)e->world * 8,
                                                cudaMemcpyHostToDevice, s),
                                "peer columns")))
            return st;
        gj.peer_maps = e->d_peer;
        gj.peer_col = (const long long *)(e->d_peer + 8 * 128);
        gj.npeer = e->world;
    }
    if (lp->gemm == CONV_GEMM_FFMA)
        st = launch_result(fc_launch_gemm_ffma(gj, V, U, Xj, s), "NK3 FFMA contraction (element shard)");
    else if (gj.vf16)
        st = launch_result(fc_launch_gemm_tcgen05_f16(gj, V, Vlo, U, Xj, s), "NK3 F16X3 contraction (element shard)");
    else
        st = launch_result(fc_launch_gemm_tcgen05(gj, V, Vlo, U, Xj, s), "NK3 3xTF32 contraction (element shard)");
    if (st || fuse_x) return st;
    // pack X_j [Xz_j][Xm][bn_tot] -> peer k: [Xz_j][Xm][bnpad_k] (its images' columns), into
    // the send buffer or straight into peer k's receive buffer at this rank's segment
    char *dst = (char *)x_send;
    long long col0 = 0;
    for (int k = 0; k < e->world; ++k) {
        const size_t wbytes = (size_t)e->bnpad[k] * 4;
        if (x_recv_peer) dst = (char *)x_recv_peer[k] + eshard_x_recv_off(e, k, e->rank);
        st = launch_result(cudaMemcpy2DAsync(dst, wbytes, (const char *)Xj + col0 * 4, (size_t)e->bn_tot * 4, wbytes,
                                             (size_t)gj.Xz * gj.Xm, cudaMemcpyDeviceToDevice, s),
                           "X pack");
        if (st) return st;
        dst += e->x_send[k];
        col0 += e->bnpad[k];
    }
    return CONV_OK;
}

conv_status conv_eshard_forward_b(conv_eshard_t e, const void *u_recv, const float *umax_all, void *x_send, void *ws,
                                  size_t ws_bytes, void *stream) {
    return eshard_forward_b_impl(e, u_recv, umax_all, x_send, nullptr, ws, ws_bytes, stream);
}

conv_status conv_eshard_forward_b_peer(conv_eshard_t e, const void *u_recv, const float *umax_all,
                                       void *const *x_recv_peer, void *ws, size_t ws_bytes, void *stream) {
    if (!x_recv_peer) {
        fc_set_error("NULL x_recv_peer array");
        return CONV_ERR_INVALID_ARG;
    }
    return eshard_forward_b_impl(e, u_recv, umax_all, nullptr, x_recv_peer, ws, ws_bytes, stream);
}

// Inter-process exchange buffers: device memory from cudaMalloc (so an IPC handle covers the
// buffer from its first byte) and its handle; a peer process maps it with conv_ipc_open.
conv_status conv_ipc_alloc(size_t bytes, void **ptr, void *handle_out) {
    if (!ptr || !handle_out || bytes == 0) {
        fc_set_error("conv_ipc_alloc: NULL argument or zero size");
        return CONV_ERR_INVALID_ARG;
    }
    *ptr = nullptr;
    cudaError_t ce = cudaMalloc(ptr, bytes);
    if (ce == cudaSuccess) ce = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t *>(handle_out), *ptr);
    if (ce != cudaSuccess) {
        if (*ptr) cudaFree(*ptr);
        *ptr = nullptr;
        fc_set_error("conv_ipc_alloc: %s", cudaGetErrorString(ce));
        return ce == cudaErrorMemoryAllocation ? CONV_ERR_OUT_OF_MEMORY : CONV_ERR_CUDA;
    }
    return CONV_OK;
}

conv_status conv_ipc_free(void *ptr) {
    if (!ptr) return CONV_OK;
    const cudaError_t ce = cudaFree(ptr);
    if (ce != cudaSuccess) {
        fc_set_error("conv_ipc_free: %s", cudaGetErrorString(ce));
        return CONV_ERR_CUDA;
    }
    return CONV_OK;
}

conv_status conv_ipc_open(const void *handle, void **ptr) {
    if (!handle || !ptr) {
        fc_set_error("conv_ipc_open: NULL argument");
        return CONV_ERR_INVALID_ARG;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    const cudaError_t ce = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (ce != cudaSuccess) {
        *ptr = nullptr;
        fc_set_error("conv_ipc_open: %s", cudaGetErrorString(ce));
        return CONV_ERR_CUDA;
    }
    return CONV_OK;
}

conv_status conv_ipc_close(void *ptr) {
    if (!ptr) return CONV_OK;
    const cudaError_t ce = cudaIpcCloseMemHandle(ptr);
    if (ce != cudaSuccess) {
        fc_set_error("conv_ipc_close: %s", cudaGetErrorString(ce));
        return CONV_ERR_CUDA;
    }
    return CONV_OK;
}

conv_status conv_eshard_forward_c(conv_eshard_t e, const void *x_recv, float *out, void *ws, size_t ws_bytes,
                                  void *stream) {
    conv_status st = eshard_check(e, ws, ws_bytes);
    if (st) return st;
    if ((st = check_dev_ptr(e->lp, x_recv, "x_recv")) || (st = check_dev_ptr(e->lp, out, "out"))) return st;
    cudaStream_t s = (cudaStream_t)stream;
    char *b = (char *)ws;
    conv_plan_s *lp = e->lp;
    const Geometry &g = lp->g;
    // peer j's chunk [px][E_j][Xm][BN_me] -> X_local rows (p E + e0_j ..) of [Xz][Xm][BN_me]
    const size_t slab = (size_t)g.Xm * g.BN_pad * 4;  // one element plane of X_local
    const char *src = (const char *)x_recv;
    for (int j = 0; j < e->world; ++j) {
        const int Ej = e->ecnt[j];
        for (int p = 0; p < e->px; ++p) {
            st = launch_result(cudaMemcpyAsync(b + e->off_X + (size_t)(p * g.E + e->elo[j]) * slab,
                                               src + (size_t)p * Ej * slab, (size_t)Ej * slab,
                                               cudaMemcpyDeviceToDevice, s),
                               "X unpack");
            if (st) return st;
        }
        src += e->x_recv[j];
    }
    return run_stage(&e->lpx, g, 3, nullptr, nullptr, out, b, s);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Backward passes (not in the paper, which times forward layers).
// Both gradients of Eq. 5 are themselves valid cross-correlations, so they run through the
// same fast forward pipeline after a re-layout of their operands (backward.cu kernels):
//   data    dX[b][c][y][x] = sum_{c'} sum_{p,q} dY[b][c'][y-p][x-q] W[c'][c][p][q]
//           = forward( pad_{r-1}(dY) as [B][C'][H+r-1][W+r-1],  Wf[c][c'][p][q] =
//             W[c'][c][r-1-p][r-1-q] ),  any method / tile of the forward plan
//   filter  dW[c'][c][p][q] = sum_b sum_{i,j} dY[b][c'][i][j] X[b][c][i+p][j+q]
//           = forward( X^T [C][B][H][W] (images <-> channels),  dY^T [C'][B][Ho][Wo] as an
//             Ho x Wo (non-isotropic) kernel ) = [C][C'][r][r], transposed to [C'][C][r][r];
//             FFT tiles of the whole image (t = H, W <= 64; conv_plan_nd) or the direct path
// ---------------------------------------------------------------------------
cudaError_t fc_launch_pad(const float *src, float *dst, long long planes, int h, int w, int pad, cudaStream_t s);
cudaError_t fc_launch_flip_transpose(const float *w, float *wf, int Cout, int C, int r, cudaStream_t s);
cudaError_t fc_launch_swap01(const float *src, float *dst, int A, int B, long long inner, cudaStream_t s);

extern "C" {

conv_status conv_plan_backward(conv_plan_t *out, int which, int B, int C, int Cout, int H, int W, int r,
                               conv_method method, int m, const conv_plan_options *opts) {
    if (!out || (which != 1 && which != 2)) {
        fc_set_error("conv_plan_backward: NULL plan pointer or which not 1 (data) / 2 (filter)");
        return CONV_ERR_INVALID_ARG;
    }
    if (B < 1 || C < 1 || Cout < 1 || r < 1 || H < r || W < r) {
        fc_set_error("sizes must be >= 1 and H, W >= r");
        return CONV_ERR_INVALID_ARG;
    }
    const int Ho = H - r + 1, Wo = W - r + 1;
    conv_plan_t inner = nullptr;
    conv_status st;
    if (which == 1) {
        st = plan_create(&inner, 0, B, Cout, C, H + r - 1, W + r - 1, r, method, m, nullptr, nullptr, nullptr, opts);
    } else {
        if (method == CONV_WINOGRAD) {
            fc_set_error("backward filter: the Ho x Wo kernel exceeds Winograd's t <= 8; use an FFT or direct method");
            return CONV_ERR_UNSUPPORTED;
        }
        const int in[2] = {H, W}, k[2] = {Ho, Wo}, mt[2] = {r, r};
        st = plan_create(&inner, 2, C, B, Cout, 0, 0, 0, method, 0, in, k, mt, opts);
    }
    if (st) return st;
    conv_plan_s *p = (conv_plan_s *)calloc(1, sizeof(conv_plan_s));
    if (!p) {
        conv_destroy(inner);
        return CONV_ERR_OUT_OF_MEMORY;
    }
    p->kind = which;
    p->inner = inner;
    p->g = inner->g;
    p->info = inner->info;
    p->device = inner->device;
    p->gemm = inner->gemm;
    const size_t a = which == 1 ? (size_t)B * Cout * (H + r - 1) * (size_t)(W + r - 1) * 4   // padded dY
                                : (size_t)B * C * (size_t)H * W * 4;                         // X^T
    const size_t b = which == 1 ? (size_t)Cout * C * r * r * 4                                 // flipped W
                                : (size_t)B * Cout * (size_t)Ho * Wo * 4;                     // dY^T
    p->off_a = 0;
    p->off_b = align256(a);
    const size_t extra = align256(a) + align256(b) + (which == 2 ? align256((size_t)C * Cout * r * r * 4) : 0);
    p->ws_bytes = extra + inner->ws_bytes;
    p->info.workspace_bytes = p->ws_bytes;
    *out = p;
    return CONV_OK;
}

static conv_status backward_check(conv_plan_s *p, int which, void *ws, size_t ws_bytes) {
    if (!p || p->kind != which) {
        fc_set_error(which == 1 ? "not a backward-data plan" : "not a backward-filter plan");
        return CONV_ERR_INVALID_ARG;
    }
    conv_status st = check_device(p);
    if (st) return st;
    if (ws_bytes < p->ws_bytes) {
        fc_set_error("workspace %zu bytes < required %zu", ws_bytes, p->ws_bytes);
        return CONV_ERR_INVALID_ARG;
    }
    return check_dev_ptr(p, ws, "workspace");
}

conv_status conv_backward_data(conv_plan_t p, const float *dy, const float *w, float *dx, void *ws, size_t ws_bytes,
                               void *stream) {
    conv_status st = backward_check(p, 1, ws, ws_bytes);
    if (st) return st;
    if ((st = check_dev_ptr(p, dy, "dy")) || (st = check_dev_ptr(p, w, "weights")) || (st = check_dev_ptr(p, dx, "dx")))
        return st;
    cudaStream_t s = (cudaStream_t)stream;
    const Geometry &g = p->inner->g;  // forward on (B, C', C, H + r - 1, W + r - 1, r)
    char *b = (char *)ws;
    float *dyp = (float *)(b + p->off_a), *wf = (float *)(b + p->off_b);
    const int r = g.r;
    if ((st = launch_result(fc_launch_pad(dy, dyp, (long long)g.B * g.C, g.H - 2 * (r - 1), g.W - 2 * (r - 1), r - 1, s),
                            "pad dY")))
        return st;
    if ((st = launch_result(fc_launch_flip_transpose(w, wf, g.C, g.Cout, r, s), "flip / transpose W"))) return st;
    const size_t extra = p->ws_bytes - p->inner->ws_bytes;
    return forward_impl(p->inner, dyp, wf, dx, b + extra, s, nullptr);
}

conv_status conv_backward_filter(conv_plan_t p, const float *x, const float *dy, float *dw, void *ws,
                                 size_t ws_bytes, void *stream) {
    conv_status st = backward_check(p, 2, ws, ws_bytes);
    if (st) return st;
    if ((st = check_dev_ptr(p, x, "x")) || (st = check_dev_ptr(p, dy, "dy")) || (st = check_dev_ptr(p, dw, "dw")))
        return st;
    cudaStream_t s = (cudaStream_t)stream;
    const Geometry &g = p->inner->g;  // forward on (B' = C, C' = B, Cout, H x W, kernel Ho x Wo)
    char *b = (char *)ws;
    float *xt = (float *)(b + p->off_a), *dyt = (float *)(b + p->off_b);
    const int C = g.B, Bn = g.C, Cout = g.Cout;
    const int H = g.ax_in[1], W = g.ax_in[2], Ho = g.ax_r[1], Wo = g.ax_r[2], r = H - Ho + 1;
    if ((st = launch_result(fc_launch_swap01(x, xt, Bn, C, (long long)H * W, s), "X^T"))) return st;
    if ((st = launch_result(fc_launch_swap01(dy, dyt, Bn, Cout, (long long)Ho * Wo, s), "dY^T"))) return st;
    const size_t extra = p->ws_bytes - p->inner->ws_bytes;
    float *dwt = (float *)(b + extra - align256((size_t)C * Cout * r * r * 4));  // [C][C'][r][r]
    if ((st = forward_impl(p->inner, xt, dyt, dwt, b + extra, s, nullptr))) return st;
    return launch_result(fc_launch_swap01(dwt, dw, C, Cout, (long long)r * r, s), "dW transpose");
}

}  // extern "C"
