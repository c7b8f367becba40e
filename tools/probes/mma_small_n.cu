// Microbenchmark: sustained tcgen05.mma kind::tf32 cost per instruction at small N (the fused
// F(2,3) kernel's M128 x N16/N32 x K8 shapes), A from shared memory (SS) or tensor memory (TS),
// accumulating into one D (dependent chain) or round-robin over 4 / 16 D's.
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/msn tools/probes/mma_small_n.cu
#include <cstdio>
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

template <int N, int TS, int ND, int NW = 1>
__global__ void k(long long *cycles, int iters) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float *>(smem)[i] = 0.f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    if (threadIdx.x % 32 == 0 && warp < NW) {
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((128u >> 4) << 24);
        const uint64_t ad = make_desc(smem_u32(smem), 16, 256, 6);
        const uint64_t bd = make_desc(smem_u32(smem + 32768), 16, 256, 6);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t d = tmem + (uint32_t)((((i % ND) * NW + warp) % 16) * N);
            if (TS)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                             "r"(tmem + 448u), "l"(bd), "r"(idesc), "r"(i)
                             : "memory");
            else
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
                             "l"(ad), "l"(bd), "r"(idesc), "r"(i)
                             : "memory");
        }
        if (warp == 0) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&bar))
                     : "memory");
        if (warp == 0) asm volatile(
            "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(
                smem_u32(&bar))
            : "memory");
        if (warp == 0) cycles[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, int TS, int ND, int NW = 1>
void run(const char *name) {
    long long *d;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaFuncSetAttribute(k<N, TS, ND, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int iters = 8192;
    k<N, TS, ND, NW><<<148, 128, 70 * 1024>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-34s err=%s cyc/mma=%.1f (ideal %d)\n", name, cudaGetErrorString(e), (double)h[0] / iters / NW, 128 * N / 256);
    cudaFree(d);
}

int main() {
    run<16, 0, 1>("SS N16 one D");
    run<16, 0, 4>("SS N16 4 D");
    run<16, 1, 1>("TS N16 one D");
    run<16, 1, 4>("TS N16 4 D");
    run<16, 1, 16>("TS N16 16 D");
    run<32, 0, 1>("SS N32 one D");
    run<32, 0, 4>("SS N32 4 D");
    run<64, 0, 4>("SS N64 4 D");
    run<128, 0, 2>("SS N128 2 D");
    run<16, 1, 4, 2>("TS N16 2 issuing warps");
    run<16, 1, 4, 4>("TS N16 4 issuing warps");
    run<32, 0, 4, 4>("SS N32 4 issuing warps");
    return 0;
}
