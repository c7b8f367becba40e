// NK3 FFMA fallback: the element-wise stage as Z batched real products
//     X_z [M x BN] = V_z [M x K] . U_z [K x BN]        (Eq. 8)
// on CUDA-core FP32 FMAs, 64x64 output tiles, 4x4 per thread, K-steps of 16.
// This is the baseline the tcgen05 3xTF32 kernel is measured against.
//
// Also NK5, the direct-convolution check path (north_star step (4); Eq. 5):
// out[b][c'][y][x] = sum_c sum_p sum_q in[b][c][y+p][x+q] w[c'][c][p][q].
#include "common.h"

namespace {

constexpr int BM = 64, BNT = 64, BK = 16;

__global__ void __launch_bounds__(256) nk3_gemm_ffma(const float *__restrict__ A, const float *__restrict__ Bm,
                                                     float *__restrict__ X, int M, int K, int lda, long long NP,
                                                     int Zn) {
    __shared__ float As[BK][BM + 4];
    __shared__ __align__(16) float Bs[BK][BNT];
    const int z = blockIdx.z;
    const int m0 = blockIdx.y * BM;
    const long long n0 = (long long)blockIdx.x * BNT;
    const float *Az = A + (size_t)z * M * lda;
    float *Xz = X + (size_t)z * M * NP;
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += BK) {
        for (int i = tid; i < BM * BK; i += 256) {
            const int row = i / BK, kk = i % BK;
            const int gm = m0 + row, gk = k0 + kk;
            As[kk][row] = (gm < M && gk < K) ? Az[(size_t)gm * lda + gk] : 0.f;
        }
        for (int i = tid; i < BK * BNT; i += 256) {
            const int kk = i / BNT, col = i % BNT;
            const int gk = k0 + kk;
            const long long gn = n0 + col;
            // U blocked by FC_TB tiles: U[n / TB][z][k][n % TB]
            Bs[kk][col] = (gk < K && gn < NP)
                              ? Bm[(((size_t)(gn / FC_TB) * Zn + z) * K + gk) * FC_TB + (size_t)(gn % FC_TB)]
                              : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
            const float4 bv = *reinterpret_cast<const float4 *>(&Bs[kk][tx * 4]);
            b[0] = bv.x; b[1] = bv.y; b[2] = bv.z; b[3] = bv.w;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int gm = m0 + ty * 4 + i;
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const long long gn = n0 + tx * 4 + j;
            if (gn < NP) Xz[(size_t)gm * NP + gn] = acc[i][j];
        }
    }
}

// NK5: CTA = 16x16 output pixels x 8 output channels of one image.
constexpr int DT = 16, DCO = 8;

__global__ void __launch_bounds__(256) nk5_direct(Geometry g, const float *__restrict__ in,
                                                  const float *__restrict__ w, float *__restrict__ out) {
    extern __shared__ float smem[];
    const int r = g.r, P = DT + r - 1;
    float *s_in = smem;            // [P][P]
    float *s_w = smem + P * P;     // [DCO][r][r]
    const int tiles_x = (g.Wo + DT - 1) / DT;
    const int by = blockIdx.x / tiles_x, bx = blockIdx.x % tiles_x;
    const int co0 = blockIdx.y * DCO, b = blockIdx.z;
    const int tx = threadIdx.x % DT, ty = threadIdx.x / DT;
    const int y0 = by * DT, x0 = bx * DT;
    float acc[DCO] = {};
    for (int c = 0; c < g.C; ++c) {
        const float *img = in + ((size_t)b * g.C + c) * g.H * g.W;
        for (int i = threadIdx.x; i < P * P; i += 256) {
            const int yy = y0 + i / P, xx = x0 + i % P;
            s_in[i] = (yy < g.H && xx < g.W) ? img[(size_t)yy * g.W + xx] : 0.f;
        }
        for (int i = threadIdx.x; i < DCO * r * r; i += 256) {
            const int k = i / (r * r), pq = i % (r * r);
            s_w[i] = (co0 + k < g.Cout) ? w[((size_t)(co0 + k) * g.C + c) * r * r + pq] : 0.f;
        }
        __syncthreads();
        for (int p = 0; p < r; ++p)
            for (int q = 0; q < r; ++q) {
                const float v = s_in[(ty + p) * P + tx + q];
#pragma unroll
                for (int k = 0; k < DCO; ++k) acc[k] = fmaf(v, s_w[(k * r + p) * r + q], acc[k]);
            }
        __syncthreads();
    }
    const int y = y0 + ty, x = x0 + tx;
    if (y < g.Ho && x < g.Wo)
#pragma unroll
        for (int k = 0; k < DCO; ++k)
            if (co0 + k < g.Cout) out[(((size_t)b * g.Cout + co0 + k) * g.Ho + y) * g.Wo + x] = acc[k];
}

// NK5, register-blocked (compile-time r = 3, 5): a CTA computes 64 output channels x an 8 x 16
// output block of one image; each of the 256 threads holds 4 channels x 8 consecutive pixels
// (32 accumulators).  Input channels are staged CK at a time in shared memory -- the (8+R-1) x
// (16+R-1) input patch with a 33-float row pitch (the 16 pixel groups of a warp hit distinct
// banks) and the weights as [c][p q][c'] so a thread's 4 channels are one 16-byte load -- with
// the next stage's global loads issued into registers before the current stage's FMAs.  Per
// (c, p) a thread loads the 8+R-1 inputs of its row once and reuses them for every q:
// 4 R^2 x 8 FMAs per (R (8+R-1) + R^2) shared loads.  Same summation order as nk5_direct
// ((c, p, q) sequential per output), so the two agree bit for bit.
constexpr int RB_CO = 64, RB_H = 8, RB_W = 16, RB_SP = 33;

template <int R, int RB_CK = (R <= 3 ? 4 : 2)>
__global__ void __launch_bounds__(256) nk5_direct_rb(Geometry g, const float *__restrict__ in,
                                                     const float *__restrict__ w, float *__restrict__ out) {
    constexpr int PH = RB_H + R - 1, PW = RB_W + R - 1;
    constexpr int IN_STAGE = RB_CK * PH * RB_SP, W_STAGE = RB_CK * R * R * RB_CO;
    constexpr int IN_LD = (RB_CK * PH * PW + 255) / 256, W_LD = (RB_CK * R * R * RB_CO + 255) / 256;
    __shared__ __align__(16) float s_in[2][IN_STAGE];
    __shared__ __align__(16) float s_w[2][W_STAGE];
    const int tiles_x = (g.Wo + RB_W - 1) / RB_W;
    const int ty0 = (blockIdx.x / tiles_x) * RB_H, tx0 = (blockIdx.x % tiles_x) * RB_W;
    const int co0 = blockIdx.y * RB_CO, b = blockIdx.z;
    const int tid = threadIdx.x, pg = tid & 15, cg = tid >> 4;
    const int row = pg >> 1, xh = (pg & 1) * 8;
    float acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    float rin[IN_LD], rw[W_LD];
    auto gload = [&](int c0) {  // stage c0 .. c0 + CK - 1 into registers (zero outside)
#pragma unroll
        for (int k = 0; k < IN_LD; ++k) {
            const int i = tid + 256 * k;
            float v = 0.f;
            if (i < RB_CK * PH * PW) {
                const int cc = i / (PH * PW), rem = i - cc * PH * PW, yy = rem / PW, xx = rem - yy * PW;
                const int c = c0 + cc, gy = ty0 + yy, gx = tx0 + xx;
                if (c < g.C && gy < g.H && gx < g.W) v = __ldg(in + (((size_t)b * g.C + c) * g.H + gy) * g.W + gx);
            }
            rin[k] = v;
        }
#pragma unroll
        for (int k = 0; k < W_LD; ++k) {
            const int i = tid + 256 * k;  // i = co * (CK R^2) + cc * R^2 + pq: runs of CK R^2 floats per c'
            float v = 0.f;
            if (i < RB_CK * R * R * RB_CO) {
                const int co = i / (RB_CK * R * R), rem = i - co * RB_CK * R * R;
                const int cc = rem / (R * R), pq = rem - cc * R * R;
                if (co0 + co < g.Cout && c0 + cc < g.C) v = __ldg(w + ((size_t)(co0 + co) * g.C + c0 + cc) * (R * R) + pq);
            }
            rw[k] = v;
        }
    };
    auto sstore = [&](int buf) {
#pragma unroll
        for (int k = 0; k < IN_LD; ++k) {
            const int i = tid + 256 * k;
            if (i < RB_CK * PH * PW) {
                const int cc = i / (PH * PW), rem = i - cc * PH * PW, yy = rem / PW, xx = rem - yy * PW;
                s_in[buf][(cc * PH + yy) * RB_SP + xx] = rin[k];
            }
        }
#pragma unroll
        for (int k = 0; k < W_LD; ++k) {
            const int i = tid + 256 * k;
            if (i < RB_CK * R * R * RB_CO) {
                const int co = i / (RB_CK * R * R), rem = i - co * RB_CK * R * R;
                const int cc = rem / (R * R), pq = rem - cc * R * R;
                s_w[buf][(cc * R * R + pq) * RB_CO + co] = rw[k];
            }
        }
    };
    gload(0);
    sstore(0);
    __syncthreads();
    const int nst = (g.C + RB_CK - 1) / RB_CK;
    for (int st = 0; st < nst; ++st) {
        const int buf = st & 1;
        if (st + 1 < nst) gload((st + 1) * RB_CK);
#pragma unroll
        for (int cc = 0; cc < RB_CK; ++cc) {
#pragma unroll
            for (int p = 0; p < R; ++p) {
                float x[8 + R - 1];
                const float *src = s_in[buf] + (cc * PH + row + p) * RB_SP + xh;
#pragma unroll
                for (int j = 0; j < 8 + R - 1; ++j) x[j] = src[j];
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    const float4 wv = *reinterpret_cast<const float4 *>(s_w[buf] + (cc * R * R + p * R + q) * RB_CO +
                                                                        cg * 4);
                    const float wr[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(x[j + q], wr[i], acc[i][j]);
                }
            }
        }
        if (st + 1 < nst) {
            __syncthreads();  // every thread is done with buf ^ 1 (read two stages ago)
            sstore(buf ^ 1);
            __syncthreads();
        }
    }
    const int y = ty0 + row;
    if (y >= g.Ho) return;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int co = co0 + cg * 4 + i;
        if (co >= g.Cout) continue;
        float *dst = out + (((size_t)b * g.Cout + co) * g.Ho + y) * g.Wo + tx0 + xh;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (tx0 + xh + j < g.Wo) dst[j] = acc[i][j];
    }
}

}  // namespace

cudaError_t fc_launch_gemm_ffma(const Geometry &g, const float *V, const float *U, float *X, cudaStream_t s) {
    dim3 grid((unsigned)((g.BN_pad + BNT - 1) / BNT), (unsigned)((g.M + BM - 1) / BM), (unsigned)g.Z);
    nk3_gemm_ffma<<<grid, 256, 0, s>>>(V, U, X, g.M, g.K, g.Kp, g.BN_pad, g.Z);
    return cudaGetLastError();
}

cudaError_t fc_launch_direct(const Geometry &g, const float *in, const float *w, float *out, cudaStream_t s) {
    if (g.r == 3 || g.r == 5) {  // register-blocked kernel
        const int tiles = ((g.Ho + RB_H - 1) / RB_H) * ((g.Wo + RB_W - 1) / RB_W);
        dim3 grid((unsigned)tiles, (unsigned)((g.Cout + RB_CO - 1) / RB_CO), (unsigned)g.B);
        if (g.r == 3)
            nk5_direct_rb<3><<<grid, 256, 0, s>>>(g, in, w, out);
        else
            nk5_direct_rb<5><<<grid, 256, 0, s>>>(g, in, w, out);
        return cudaGetLastError();
    }
    const int P = DT + g.r - 1;
    const size_t smem = sizeof(float) * ((size_t)P * P + (size_t)DCO * g.r * g.r);
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    fc_smem_attr((const void *)nk5_direct, 200 * 1024);
    const int tiles = ((g.Ho + DT - 1) / DT) * ((g.Wo + DT - 1) / DT);
    dim3 grid((unsigned)tiles, (unsigned)((g.Cout + DCO - 1) / DCO), (unsigned)g.B);
    nk5_direct<<<grid, 256, smem, s>>>(g, in, w, out);
    return cudaGetLastError();
}
