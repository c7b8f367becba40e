// Microbenchmark: sustained tcgen05.mma kind::tf32 issue rate for operand layouts
// used by NK3 (cycles per instruction, one CTA per SM, operands resident in smem).
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

template <int N, int BMAJ, int KIND>  // KIND 0 = tf32, 1 = bf16 (f16 kind)
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
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t fmt = KIND == 0 ? 2u : 1u;
        const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)BMAJ << 16) | ((N >> 3) << 17) |
                               ((128u >> 4) << 24);
        const uint32_t A = smem_u32(smem), B = smem_u32(smem + 32768);
        const uint64_t ad = make_desc(A, 16, 1024, 2);
        const uint64_t bd = BMAJ ? make_desc(B, 4096, 512, 1) : make_desc(B, 16, 1024, 2);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (KIND == 0)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                             "l"(ad), "l"(bd), "r"(idesc), "r"(i)
                             : "memory");
            else
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                             "l"(ad), "l"(bd), "r"(idesc), "r"(i)
                             : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&bar))
                     : "memory");
        asm volatile(
            "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(
                smem_u32(&bar))
            : "memory");
        cycles[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

template <int N, int BMAJ, int KIND>
void run(const char *name) {
    long long *d;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaFuncSetAttribute(k<N, BMAJ, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int iters = 4096;
    k<N, BMAJ, KIND><<<148, 128, 70 * 1024>>>(d, iters);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<N, BMAJ, KIND><<<148, 128, 70 * 1024>>>(d, iters);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const double kk = KIND == 0 ? 8 : 16;
    const double flops = 2.0 * 128 * N * kk * iters * 148;
    printf("%-28s err=%s cyc/mma=%.1f  TFLOP/s=%.1f\n", name, cudaGetErrorString(e), (double)h[0] / iters,
           flops / (ms * 1e-3) / 1e12);
    cudaFree(d);
}

int main() {
    run<256, 0, 0>("tf32 N256 B K-major");
    run<256, 1, 0>("tf32 N256 B MN-major 32B");
    run<128, 0, 0>("tf32 N128 B K-major");
    run<128, 1, 0>("tf32 N128 B MN-major 32B");
    run<256, 0, 1>("bf16 N256 B K-major");
    return 0;
}
