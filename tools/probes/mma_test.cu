// Numeric check of tcgen05 kind::tf32 with A K-major SW128 and B MN-major SW128_BASE32B.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
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

constexpr int M = 128, N = 128, K = 8;

__global__ void k(const float *Ag, const float *Bg, float *out, int lbo, int sbo) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    uint8_t *A = smem;            // 128 rows x 128 B (only first 32 B per row used for K=8)
    uint8_t *B = smem + 16384;    // 4 blocks of 32 n x 8 k
    for (int i = threadIdx.x; i < M * K; i += blockDim.x) {
        const int m = i / K, kk = i % K;
        const int off = m * 128 + (((kk / 4) ^ (m % 8)) * 16) + (kk % 4) * 4;
        *reinterpret_cast<float *>(A + off) = Ag[m * K + kk];
    }
    for (int i = threadIdx.x; i < K * N; i += blockDim.x) {
        const int kk = i / N, n = i % N, nb = n / 32, nn = n % 32;
        const int off = nb * lbo + kk * 128 + (((nn / 8) ^ (kk % 4)) * 32) + (nn % 8) * 4;
        *reinterpret_cast<float *>(B + off) = Bg[kk * N + n];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
        const uint64_t ad = make_desc(smem_u32(A), 16, 1024, 2);
        const uint64_t bd = make_desc(smem_u32(B), lbo, sbo, 1);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"(0)
            : "memory");
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
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

int main() {
    static float hA[M * K], hB[K * N], hD[M * N];
    for (int i = 0; i < M * K; ++i) hA[i] = (float)((i * 7) % 13 - 6);
    const bool trunc_test = getenv("TRUNC") != nullptr;
    if (trunc_test) { for (int i = 0; i < M * K; ++i) hA[i] = 1.0f + 3.0f / 4096.0f; }
    for (int i = 0; i < K * N; ++i) hB[i] = trunc_test ? 1.0f : (float)((i * 5) % 11 - 5);
    float *dA, *dB, *dD;
    cudaMalloc(&dA, sizeof(hA));
    cudaMalloc(&dB, sizeof(hB));
    cudaMalloc(&dD, sizeof(hD));
    cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const int cfg[2][2] = {{1024, 512}, {512, 1024}};
    for (int v = 0; v < 2; ++v) {
        cudaMemset(dD, 0, sizeof(hD));
        k<<<1, 128, 40 * 1024>>>(dA, dB, dD, cfg[v][0], cfg[v][1]);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(hD, dD, sizeof(hD), cudaMemcpyDeviceToHost);
        int bad = 0;
        double maxerr = 0;
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                double ref = 0;
                for (int kk = 0; kk < K; ++kk) ref += (double)hA[m * K + kk] * hB[kk * N + n];
                double d = hD[m * N + n] - ref;
                if (d != 0) ++bad;
                if (d < 0) d = -d;
                if (d > maxerr) maxerr = d;
            }
        printf("lbo=%d sbo=%d err=%s bad=%d maxerr=%g D[0][0..3]=%g %g %g %g\n", cfg[v][0], cfg[v][1],
               cudaGetErrorString(e), bad, maxerr, hD[0], hD[1], hD[2], hD[3]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
