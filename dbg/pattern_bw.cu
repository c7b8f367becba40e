// Bandwidth of the NK2/NK4 access patterns in isolation (no arithmetic):
//  (a) plain copy, (b) U-style stores: each thread writes E floats at stride
//  estride (lanes contiguous along n), (c) X-style loads with the same pattern.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void copy_k(const float4 *__restrict__ a, float4 *__restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

template <int E>
__global__ void scatter_store(float *__restrict__ U, long long BN, size_t estride, int C) {
    const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (n >= BN) return;
    float *p = U + (size_t)c * BN + n;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        *p = (float)e;
        p += estride;
    }
}

template <int E>
__global__ void gather_load(const float *__restrict__ X, float *__restrict__ out, long long BN, size_t estride) {
    const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (n >= BN) return;
    const float *p = X + (size_t)c * BN + n;
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        s += __ldcs(p);
        p += estride;
    }
    if (s == 12345.f) out[n] = s;
}

int main() {
    const long long BN = 12544;  // VGG-3.2 F(4,3): 64 images x 196 tiles
    const int C = 256;
    constexpr int E = 36;
    const size_t estride = (size_t)C * BN;
    const size_t total = estride * E;  // 462 MB
    float *U, *X, *out;
    cudaMalloc(&U, total * 4);
    cudaMalloc(&X, total * 4);
    cudaMalloc(&out, BN * 4);
    cudaMemset(X, 0, total * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        copy_k<<<148 * 8, 512>>>((const float4 *)X, (float4 *)U, total / 4);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("copy          %.1f us  %.0f GB/s\n", ms * 1e3, 2.0 * total * 4 / (ms * 1e-3) / 1e9);
        for (int bs : {128, 256}) {
            cudaEventRecord(a);
            scatter_store<E><<<dim3((unsigned)((BN + bs - 1) / bs), C), bs>>>(U, BN, estride, C);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("scatter bs=%d %.1f us  %.0f GB/s\n", bs, ms * 1e3, 1.0 * total * 4 / (ms * 1e-3) / 1e9);
            cudaEventRecord(a);
            gather_load<E><<<dim3((unsigned)((BN + bs - 1) / bs), C), bs>>>(X, out, BN, estride);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("gather  bs=%d %.1f us  %.0f GB/s\n", bs, ms * 1e3, 1.0 * total * 4 / (ms * 1e-3) / 1e9);
        }
    }
    printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
