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

}  // namespace

cudaError_t fc_launch_gemm_ffma(const Geometry &g, const float *V, const float *U, float *X, cudaStream_t s) {
    dim3 grid((unsigned)((g.BN_pad + BNT - 1) / BNT), (unsigned)((g.M + BM - 1) / BM), (unsigned)g.Z);
    nk3_gemm_ffma<<<grid, 256, 0, s>>>(V, U, X, g.M, g.K, g.Kp, g.BN_pad, g.Z);
    return cudaGetLastError();
}

cudaError_t fc_launch_direct(const Geometry &g, const float *in, const float *w, float *out, cudaStream_t s) {
    const int P = DT + g.r - 1;
    const size_t smem = sizeof(float) * ((size_t)P * P + (size_t)DCO * g.r * g.r);
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    fc_smem_attr((const void *)nk5_direct, 200 * 1024);
    const int tiles = ((g.Ho + DT - 1) / DT) * ((g.Wo + DT - 1) / DT);
    dim3 grid((unsigned)tiles, (unsigned)((g.Cout + DCO - 1) / DCO), (unsigned)g.B);
    nk5_direct<<<grid, 256, smem, s>>>(g, in, w, out);
    return cudaGetLastError();
}
