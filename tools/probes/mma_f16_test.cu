// Numeric check of tcgen05 kind::f16 (fp16 x fp16 -> fp32) with A and B both
// K-major, SWIZZLE_64B (64-byte rows = 32 fp16 of K), M=128 N=256, K=32 as two
// K=16 instructions (descriptor start +32 B), plus the A-negate bit.
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/mf16 dbg/mma_f16_test.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

constexpr int M = 128, N = 256, K = 32;

// K-major SW64: row r (64 B), 16-byte chunk c -> c ^ ((r >> 1) & 3)
__device__ __forceinline__ int sw64(int row, int k) {
    return row * 64 + ((((k >> 3) ^ (row >> 1)) & 3) << 4) + (k & 7) * 2;
}

__global__ void k(const float *Ag, const float *Bg, float *out, int negate) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    uint8_t *A = smem;               // 128 rows x 64 B = 8 KB
    uint8_t *B = smem + 8192;        // 256 rows x 64 B = 16 KB
    for (int i = threadIdx.x; i < M * K; i += blockDim.x) {
        const int m = i / K, kk = i % K;
        *reinterpret_cast<__half *>(A + sw64(m, kk)) = __float2half_rn(Ag[m * K + kk]);
    }
    for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
        const int n = i / K, kk = i % K;
        *reinterpret_cast<__half *>(B + sw64(n, kk)) = __float2half_rn(Bg[kk * N + n]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        // kind::f16: D f32 (bit 4), A/B f16 (0), both K-major, N>>3 at 17, M>>4 at 24
        uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        if (negate) idesc |= 1u << 13;
        for (int s = 0; s < 2; ++s) {
            const uint64_t ad = make_desc(smem_u32(A) + 32 * s, 16, 512, 4);
            const uint64_t bd = make_desc(smem_u32(B) + 32 * s, 16, 512, 4);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                "l"(ad), "l"(bd), "r"(idesc), "r"(s)
                : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&bar))
                     : "memory");
    }
    __syncwarp();
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(
            smem_u32(&bar))
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int c = 0; c < N; c += 4) {
        uint32_t v[4];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                     : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 4; ++j) out[threadIdx.x * N + c + j] = __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
    static float hA[M * K], hB[K * N], hD[M * N];
    for (int i = 0; i < M * K; ++i) hA[i] = (float)((i * 7) % 13 - 6) + 0.5f * ((i / 3) % 3);
    for (int i = 0; i < K * N; ++i) hB[i] = (float)((i * 5) % 11 - 5) * 0.25f;
    float *dA, *dB, *dD;
    cudaMalloc(&dA, sizeof(hA));
    cudaMalloc(&dB, sizeof(hB));
    cudaMalloc(&dD, sizeof(hD));
    cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    int rc = 0;
    for (int neg = 0; neg < 2; ++neg) {
        cudaMemset(dD, 0, sizeof(hD));
        k<<<1, 128, 40 * 1024>>>(dA, dB, dD, neg);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(hD, dD, sizeof(hD), cudaMemcpyDeviceToHost);
        int bad = 0;
        double maxerr = 0;
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                double ref = 0;
                for (int kk = 0; kk < K; ++kk) ref += (double)hA[m * K + kk] * hB[kk * N + n];
                if (neg) ref = -ref;
                double d = hD[m * N + n] - ref;
                if (d != 0) ++bad;
                if (d < 0) d = -d;
                if (d > maxerr) maxerr = d;
            }
        printf("f16 K-major SW64 negate=%d err=%s bad=%d maxerr=%g D[0][0..3]=%g %g %g %g\n", neg,
               cudaGetErrorString(e), bad, maxerr, hD[0], hD[1], hD[2], hD[3]);
        if (e != cudaSuccess || bad) rc = 1;
    }
    return rc;
}
