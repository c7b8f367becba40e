// Internal declarations shared by the fastconv CUDA translation units.
// (Product path only; nothing here is shared with oracle/.)
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include <stddef.h>

#include "../../include/fastconv.h"

#define FC_MAX_T 64          // largest FFT tile edge supported (Winograd: 8)

// Device-side constants of a plan (fp32, rounded once from fp64 / exact rationals).
// Row transform "L" is applied along tile rows (index a, the H axis) and
// "R" along columns (index b, the W axis); forward 2-D transform is
//     Y[k][l] = sum_a sum_b L[k][a] d[a][b] R[l][b]
// Winograd: L = R = B^T (Eq. 4, "B f B^T"), kernel: G, inverse: A^T.
// FFT: L[k][a] = R[k][a] = exp(-2 pi i k a / t), stored as twiddles.
struct ConvConsts {
    float BT[8 * 8];     // Winograd B^T [t][t]
    float G[8 * 8];      // Winograd G [t][r]
    float AT[8 * 8];     // Winograd A^T [m][t]
    float cosv[FC_MAX_T];  // cos(2 pi j / t), j < t   (fp64 -> fp32)
    float sinv[FC_MAX_T];  // sin(2 pi j / t)
};

// Division by a runtime constant d >= 1 for dividends n < 2^31 (Granlund-Montgomery, as in
// CUTLASS's FastDivmod): q = umulhi(n, mul) >> shift with p = 31 + ceil(log2 d),
// mul = ceil(2^p / d) < 2^32 -- two instructions instead of a ~20-instruction division.
struct FastDiv {
    unsigned int mul, shift;
    int d;
};
inline FastDiv fc_fastdiv(int d) {
    FastDiv f;
    f.d = d;
    if (d <= 1) {  // q = n (fc_div tests d == 1)
        f.mul = 0;
        f.shift = 0;
        return f;
    }
    int l = 0;
    while ((1ll << l) < d) ++l;
    const int p = 31 + l;
    f.mul = (unsigned int)(((1ull << p) + (unsigned long long)d - 1) / (unsigned long long)d);
    f.shift = (unsigned int)(p - 32);
    return f;
}
#ifdef __CUDACC__
__device__ __forceinline__ int fc_div(int n, const FastDiv &f) {
    return f.d == 1 ? n : (int)(__umulhi((unsigned)n, f.mul) >> f.shift);
}
#endif

struct Geometry {
    int B, C, Cout, H, W, r, m, method;
    int Ho, Wo, t, n_h, n_w, N, h, E, planes;
    long long BN, BN_pad;
    int Z, M, K;  // contraction batch / rows (output channels side) / reduction
    int Kp;       // row pitch of V (K rounded up to 4 floats = 16 B, for TMA)
    int cplx;     // Regular-FFT complex mode (tcgen05, C' % 256 == 0, C % 16 == 0): V stored as
                  // (V_r, V_i) planes [E][2][C'][Kp], Kp = round4(C), instead of the 4x real
                  // embedding; the contraction picks the plane per K-half and negates -V_i
    // F16X3 contraction (conv_gemm_impl CONV_GEMM_TCGEN05_F16X3): V_hi / V_lo are fp16,
    // Kp = K rounded up to 8 (16-byte rows), scaled per output channel c' by
    // vscale[c'] = 2^k (inverse at vscale[Cout + c']); NK2 reduces max|U| of every image b
    // into umax[b] (fp32 bits, [B] words, reset before every NK2), and the contraction scales
    // the columns of image b by s_u[b] = 2^(15 - e), max|U_b| < 2^e.  Pointers are filled per
    // call (workspace).
    int vf16;
    float vbound;            // host bound: max|V[.][c'][.]| <= vbound * max|W[c']|
    unsigned int *umax;      // [B] per-image max|U|, NK2 -> NK3 (nullptr: NK2 does not reduce)
    float *vscale;           // [2][Cout]: NK1 writes, NK3 epilogue reads the inverse
    FastDiv divN, divNw;     // n -> (image, tile) and tile -> (row, column) in the transforms
    // X = [Xz][Xm][BN_pad]: Xz = Z, Xm = M, except the Gauss epilogue combine (gc = 1:
    // F16X3, C' % 32 == 0), where the contraction stores Re = T1 - T3 and Im = T1 + T2
    // as rows [0, C') / [C', 2C') of Xz = E planes -- the Regular-FFT layout
    // ("X at w = 2")
    int gc, Xz, Xm;
    int tc_1sm;  // conv_plan_options.single_cta_mma: single-CTA contraction tiles even when M > 128
    // N-dimensional / non-isotropic layers (conv_plan_nd; "an arbitrary number of
    // dimensions, as well as non-isotropic kernels"): nd = 0 for the 2-D isotropic plans above;
    // nd = 1..3 runs the generic separable transforms of transforms_nd.cu.  Axis arrays are
    // right-aligned in 3 slots (slot 2 = the last, fastest axis; unused leading slots hold 1).
    int nd;
    int ax_in[3], ax_r[3], ax_m[3], ax_t[3], ax_n[3], ax_o[3];
    int ax_len[3];  // transformed length per axis: t, except the FFT's last axis t/2 + 1
    long long vin, vout;  // input / output elements per (image, channel) plane or volume
    int kvol;             // kernel elements per (c', c): r^2 (2-D) or prod r_d
    // element-sharded execution (conv_eshard_*): the generic NK1 writes only the transformed
    // elements e in [e_lo, e_hi), at z relative to e_lo (V of E' = e_hi - e_lo elements)
    int e_lo, e_hi;
    int fused;  // conv_plan_options.fused: NK2-NK4 in one kernel (fused_wino.cu)
    // element-shard peer exchange (conv_eshard_forward_b_peer): the tcgen05 contraction stores
    // each 32-column X box straight into its owner's receive buffer; device arrays of npeer
    // tensor maps and first columns (0: the plan's own X)
    const void *peer_maps;
    const long long *peer_col;
    int npeer;
};

// Per-axis constants of an N-D plan (fp64 -> fp32 once): Winograd B^T [t][t], G [t][r],
// A^T [m][t] of F(m_d, r_d), and the twiddles cos / sin(2 pi j / t_d).
struct NdConsts {
    float BT[3][64], G[3][64], AT[3][64];
    float cosv[3][FC_MAX_T], sinv[3][FC_MAX_T];
};

struct conv_plan_s {
    Geometry g;
    conv_gemm_impl gemm;
    int device;
    ConvConsts host_consts;
    double AT64[64], BT64[64], G64[64];  // exact Winograd matrices (fp64)
    ConvConsts *d_consts;                 // device copy
    NdConsts *d_nd;                       // N-D plans: per-axis constants (device)
    int generic_transforms;               // 1: force the runtime-t reference transform kernels
    size_t off_V, off_Vlo, off_U, off_X, ws_bytes;
    size_t off_vscale, off_umax;          // F16X3: per-c' scales [2][Cout], per-image max|U| [B] (else 0)
    int chunk, nchunks;                   // L2-resident batch chunking (images per chunk)
    int kind;                             // 0 forward; 1 / 2 backward data / filter (conv_plan_backward)
    conv_plan_s *inner;                   // backward plans: the forward plan they run
    size_t off_a, off_b;                  // backward plans: workspace offsets of the re-laid-out operands
    int e2e_chunks;                       // pipelining depth of conv_forward_host
    cudaStream_t h2d, d2h;                // copy streams of the pipelined host path
    // NK1 runs on `aux` concurrently with NK2 (they are independent; NK3 joins both):
    // fork / join event pairs taken round-robin per forward call (thread-safe counter)
    cudaStream_t aux;
#define FC_EVPAIRS 32
    cudaEvent_t fork_ev[FC_EVPAIRS], join_ev[FC_EVPAIRS];
    unsigned evc;
    int overlap_nk1;
    conv_plan_info info;
};

// U layout, blocked by FC_TB tiles: U[nb][z][k][t] with n = nb * FC_TB + t.  With a
// channel-fastest NK2 grid, consecutive CTAs (channels k, k+1 of one 128-tile block) write
// neighbouring 512-byte rows of every element slab, i.e. one sequential region per block;
// the contraction's (128 tiles x 32 k) box of one (z, block) is a single contiguous 16 KB
// run (4-D tensor map).  BN_pad is a multiple of FC_TB.
#define FC_TB 128
inline __host__ __device__ size_t fc_u_off(const Geometry &g, long long n, int k, int z) {
    return (((size_t)(n / FC_TB) * g.Z + z) * g.K + k) * FC_TB + (size_t)(n % FC_TB);
}
// stride (floats) between consecutive transformed elements z of one (tile, k)
inline __host__ __device__ size_t fc_u_zs(const Geometry &g) { return (size_t)g.K * FC_TB; }

// elements of V (one of V_hi / V_lo; fp32, or fp16 in F16X3 mode)
inline size_t fc_v_floats(const Geometry &g) {
    return g.cplx ? (size_t)2 * g.E * g.Cout * g.Kp : (size_t)g.Z * g.M * g.Kp;
}
inline size_t fc_v_bytes(const Geometry &g) { return fc_v_floats(g) * (g.vf16 ? 2 : 4); }

// F16X3 per-image max|U| (the contraction's U scale is per image, so an image's arithmetic
// never depends on the other images of its batch, chunk or shard): every thread of the block
// calls this once with its image b (b < 0: no contribution) and its non-negative max v.  Lanes
// of one image are combined in the warp, warps through shared slots for the 32 images starting
// at b0 (the image of the CTA's first tile), then one global atomicMax per (CTA, image) into
// umax[b] (fp32 bit patterns of non-negative floats order as unsigned integers).  Images
// outside the 32 slots fall back to one global atomic per warp.  No early returns before it.
#ifdef __CUDACC__
__device__ __forceinline__ void fc_block_umax_img(unsigned int *umax, int b0, int b, float v) {
    __shared__ unsigned int s_max[32];
    if (threadIdx.x < 32) s_max[threadIdx.x] = 0u;
    __syncthreads();
    const unsigned int grp = __match_any_sync(0xffffffffu, b);
    const unsigned int u = __reduce_max_sync(grp, __float_as_uint(v));
    if ((threadIdx.x & 31) == (unsigned)(__ffs(grp) - 1) && b >= 0 && u) {
        const int slot = b - b0;
        if (slot >= 0 && slot < 32)
            atomicMax(&s_max[slot], u);
        else
            atomicMax(umax + b, u);
    }
    __syncthreads();
    if (threadIdx.x < 32 && s_max[threadIdx.x]) atomicMax(umax + b0 + threadIdx.x, s_max[threadIdx.x]);
}
// Store one transformed-kernel value V[o]: split 0 = fp32; 1 = 3xTF32 pair
// (hi = rna_tf32(v), lo = v - hi, fp32); 2 = F16X3 pair of scaled fp16
// (x = v * sv, hi = rn_f16(x), lo = rn_f16(x - hi)).
__device__ __forceinline__ void fc_store_v(float *V, float *Vlo, size_t o, float v, int split, float sv) {
    if (split == 2) {
        const float x = v * sv;
        const __half hi = __float2half_rn(x);
        reinterpret_cast<__half *>(V)[o] = hi;
        reinterpret_cast<__half *>(Vlo)[o] = __float2half_rn(x - __half2float(hi));
    } else if (split) {  // V_lo rounded to the nearest TF32 too (the MMA would truncate it)
        uint32_t r;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
        const float hi = __uint_as_float(r);
        V[o] = hi;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v - hi));
        Vlo[o] = __uint_as_float(r);
    } else {
        V[o] = v;
    }
}
// Two adjacent values V[o], V[o+1] (o even) of the F16X3 pair as half2 stores.
__device__ __forceinline__ void fc_store_v2(float *V, float *Vlo, size_t o, float v0, float v1, float sv) {
    const float x0 = v0 * sv, x1 = v1 * sv;
    const __half2 hi = __floats2half2_rn(x0, x1);
    const float2 hf = __half22float2(hi);
    reinterpret_cast<__half2 *>(V)[o >> 1] = hi;
    reinterpret_cast<__half2 *>(Vlo)[o >> 1] = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
}
// exact power-of-two scale s (declared below)
__device__ __forceinline__ float fc_pow2_scale(float mx, int top);
// F16X3: an NK1 CTA owns one output channel c': block-wide max|W[c'][.][.][.]| (C r^2
// contiguous floats) -> s_v[c'] = 2^k with s_v * vbound * max|W| < 2^14, so every
// |V[.][c'][.]| * s_v < 2^14 < fp16 max; thread 0 records s_v and 1/s_v (exact).
// Every thread of the block must call it (once per kernel).
__device__ __forceinline__ float fc_row_vscale(const Geometry &g, const float *__restrict__ w, int co) {
    __shared__ float s_red[32];
    const int len = g.C * g.kvol;
    const float *row = w + (size_t)co * len;
    float mx = 0.f;
    // all loads of a round issued before any use (one memory round trip per 8 x blockDim x 4 floats)
    if ((((uintptr_t)row) & 15) == 0) {
        const float4 *r4 = reinterpret_cast<const float4 *>(row);
        const int n4 = len >> 2;
        for (int b = threadIdx.x; b < n4; b += 8 * blockDim.x) {
            float4 v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int i = b + j * blockDim.x;
                v[j] = i < n4 ? __ldg(r4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j)
                mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v[j].x), fabsf(v[j].y)), fmaxf(fabsf(v[j].z), fabsf(v[j].w))));
        }
        for (int i = (n4 << 2) + threadIdx.x; i < len; i += blockDim.x) mx = fmaxf(mx, fabsf(__ldg(row + i)));
    } else {
        for (int b = threadIdx.x; b < len; b += 8 * blockDim.x) {
            float v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int i = b + j * blockDim.x;
                v[j] = i < len ? __ldg(row + i) : 0.f;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) mx = fmaxf(mx, fabsf(v[j]));
        }
    }
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = 0.f;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) mx = fmaxf(mx, s_red[i]);
    const float sv = fc_pow2_scale(mx * g.vbound, 14);
    if (threadIdx.x == 0 && blockIdx.y == 0) {
        g.vscale[co] = sv;
        g.vscale[g.Cout + co] = 1.f / sv;
    }
    return sv;
}
// exact power-of-two scale s with max * s in [2^(top-1), 2^top); 1 for 0 / non-finite max
__device__ __forceinline__ float fc_pow2_scale(float mx, int top) {
    if (!(mx > 0.f) || !(mx < 3.0e38f)) return 1.f;
    int ex;
    frexpf(mx, &ex);  // mx = f 2^ex, f in [0.5, 1)
    int k = top - ex;
    k = k > 126 ? 126 : (k < -126 ? -126 : k);
    return ldexpf(1.f, k);
}
#endif

// geometry of a chunk of Bc images (U / X row pitch BN_pad follows the chunk)
Geometry fc_chunk_geometry(const Geometry &g, int Bc);

// ---- host helpers ----
// Allow `bytes` of dynamic shared memory for `func` on the current device, once per
// (kernel, device): the attribute is per device, so a process that drives several
// GPUs sets it on each (thread-safe).
cudaError_t fc_smem_attr(const void *func, int bytes);
// SM count of the current device (persistent grids)
int fc_num_sms();
// clusters of `cfg`'s shape (cluster dims, block, dynamic smem) that can be co-resident on
// the current device -- a persistent clustered grid larger than this runs in two waves
// (cached per (kernel, device); 0 if the query fails)
int fc_max_clusters(const void *func, const cudaLaunchConfig_t *cfg);
// opts: resolved options (never NULL; opts->gemm may be CONV_GEMM_AUTO for queries)
conv_status fc_fill_geometry(int B, int C, int Cout, int H, int W, int r, int method, int m,
                             Geometry *g, conv_plan_info *info, const conv_plan_options *opts);
conv_status fc_winograd_rational(int m, int r, double *AT, double *BT, double *G);
// planner (conv_plan_best_m): the stage-sum model's ms for a filled plan, and the best m
double fc_model_ms(const conv_plan_info &I, const Geometry &G);
conv_status fc_best_m(int B, int C, int Cout, int H, int W, int r, int method, const conv_plan_options *opts,
                      int *m_out, double *model_ms, int max_cand, int *n_cand, int *cand_m, double *cand_ms);
// 1 when (method, t, m, r) has compile-time-t NK2 / NK4 kernels (transforms_fast.cu)
int fc_fast_transforms(int method, int t, int m, int r);
// kernel launches NK1 issues (2 = F16X3 FFT codelets: per-c' scale prologue + transform)
int fc_nk1_launches(const Geometry &g, int split);
void fc_set_error(const char *fmt, ...);

// ---- kernel launchers (return cudaGetLastError()) ----
cudaError_t fc_launch_kernel_transform(const Geometry &g, const ConvConsts *dc, const float *w,
                                       float *V, float *Vlo, int split, cudaStream_t s);
cudaError_t fc_launch_input_transform(const Geometry &g, const ConvConsts *dc, const float *in,
                                      float *U, cudaStream_t s);
cudaError_t fc_launch_output_transform(const Geometry &g, const ConvConsts *dc, const float *X,
                                       float *out, cudaStream_t s);
cudaError_t fc_launch_gemm_ffma(const Geometry &g, const float *V, const float *U, float *X,
                                cudaStream_t s);
cudaError_t fc_launch_gemm_tcgen05(const Geometry &g, const float *Vhi, const float *Vlo,
                                   const float *U, float *X, cudaStream_t s);
// F16X3: Vhi / Vlo are fp16 planes; scales via g.vscale / g.umax
cudaError_t fc_launch_gemm_tcgen05_f16(const Geometry &g, const void *Vhi, const void *Vlo,
                                       const float *U, float *X, cudaStream_t s);
cudaError_t fc_launch_direct(const Geometry &g, const float *in, const float *w, float *out,
                             cudaStream_t s);
// N-D generic transforms (transforms_nd.cu): stage 0 = NK1, 1 = NK2, 3 = NK4; direct check path
cudaError_t fc_launch_nd_stage(const Geometry &g, const NdConsts *dc, int stage, const float *src, float *dst,
                               float *Vlo, int split, cudaStream_t s);
cudaError_t fc_launch_nd_direct(const Geometry &g, const float *in, const float *w, float *out, cudaStream_t s);
int fc_tcgen05_available();
cudaError_t fc_init_twiddles();
// FFT NK2 (forward) / NK4 transforms with compile-time t, split over fft_xforms_{a,b,c}.cu;
// *handled = 0 when that unit has no codelet for g.t
cudaError_t fc_fft_xform_a(const Geometry &g, const float *src, float *dst, bool forward, cudaStream_t s, int *handled);
cudaError_t fc_fft_xform_b(const Geometry &g, const float *src, float *dst, bool forward, cudaStream_t s, int *handled);
cudaError_t fc_fft_xform_c(const Geometry &g, const float *src, float *dst, bool forward, cudaStream_t s, int *handled);
// cuTensorMapEncodeTiled for an fp32 tensor (map: a 64-byte-aligned CUtensorMap; dims / box
// innermost first; strides_bytes: rank - 1 entries; swizzle_bytes 0, 32, 64 or 128)
bool fc_tma_encode_f32(void *map, const void *ptr, int rank, const unsigned long long *dims,
                       const unsigned long long *strides_bytes, const unsigned int *box, int swizzle_bytes);
// NK2 + NK3 + NK4 fused for Winograd F(2,3) with the 3xTF32 contraction (fused_wino.cu,
// conv_plan_options.fused): input -> output in one kernel, V from NK1
bool fc_fused_wino23_eligible(const Geometry &g);
int fc_fused_wino23_lw(int n_h, int n_w);
cudaError_t fc_launch_fused_wino23(const Geometry &g, const float *in, const float *Vhi, const float *Vlo,
                                   float *out, cudaStream_t s);
cudaError_t fc_fft_twiddles_a();
cudaError_t fc_fft_twiddles_b();
cudaError_t fc_fft_twiddles_c();

// compile-time-t transforms; *handled = 0 when t has no specialisation
cudaError_t fc_launch_kernel_transform_fast(const Geometry &g, const ConvConsts &hc, const float *w, float *V,
                                            float *Vlo, int split, cudaStream_t s, int *handled);
cudaError_t fc_launch_transform_fast(const Geometry &g, const ConvConsts &hc, const float *src, float *dst,
                                     int forward, cudaStream_t s, int *handled);
