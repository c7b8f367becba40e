// Layout check for tcgen05.mma kind::f16 with the A operand in tensor memory ("TS"):
// A written by tcgen05.st.32x32b (lane = row, column j = fp16 pair (k = 2j, 2j+1)), B K-major
// SWIZZLE_64B in shared memory; M=128 N=128 K=32 as two K=16 MMAs (A column offset +8).
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/mts dbg/mma_ts_test.cu
#include <cstdio>
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
constexpr int M = 128, N = 128, K = 32;
__device__ __forceinline__ int sw64(int row, int k) {
    return row * 64 + ((((k >> 3) ^ (row >> 1)) & 3) << 4) + (k & 7) * 2;
}
__device__ __forceinline__ uint32_t pack(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}

__global__ void k(const float *Ag, const float *Bg, float *out, int swap) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    uint8_t *B = smem;  // 128 rows x 64 B
    for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
        const int n = i / K, kk = i % K;
        *reinterpret_cast<__half *>(B + sw64(n, kk)) = __float2half_rn(Bg[kk * N + n]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
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
    const uint32_t acol = 128;
    {  // A row r = 32 warp + lane into columns acol .. acol + 15
        const int r = warp * 32 + lane;
        uint32_t v[16];
        for (int j = 0; j < 16; ++j) {
            const float a0 = Ag[r * K + 2 * j], a1 = Ag[r * K + 2 * j + 1];
            v[j] = swap ? pack(a1, a0) : pack(a0, a1);
        }
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + acol;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
                taddr),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
            "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
            : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) {
        uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        for (int s = 0; s < 2; ++s) {
            const uint64_t bd = make_desc(smem_u32(B) + 32 * s, 16, 512, 4);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem),
                "r"(tmem + acol + 8 * s), "l"(bd), "r"(idesc), "r"(s)
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
    int rc = 1;
    for (int swap = 0; swap < 2; ++swap) {
        cudaMemset(dD, 0, sizeof(hD));
        k<<<1, 128, 16 * 1024>>>(dA, dB, dD, swap);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(hD, dD, sizeof(hD), cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                double ref = 0;
                for (int kk = 0; kk < K; ++kk) ref += (double)hA[m * K + kk] * hB[kk * N + n];
                if (hD[m * N + n] != ref) ++bad;
            }
        printf("TS f16 swap=%d err=%s bad=%d D[0][0..3]=%g %g %g %g\n", swap, cudaGetErrorString(e), bad, hD[0], hD[1],
               hD[2], hD[3]);
        if (e == cudaSuccess && bad == 0) rc = 0;
    }
    return rc;
}
