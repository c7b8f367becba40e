// Re-layout kernels of the backward passes (api.cu "Backward passes"): zero padding of the
// output gradient, the flipped / channel-transposed kernel, and the swap of a 4-D tensor's
// two leading dimensions.  Pure data movement (coalesced along the innermost dimension).
#include "common.h"

namespace {

// dst[pl][y][x] = src[pl][y - pad][x - pad] inside, 0 in the border; dst is (h + 2 pad) x (w + 2 pad)
__global__ void pad_kernel(const float *__restrict__ src, float *__restrict__ dst, long long planes, int h, int w,
                           int pad) {
    const int H2 = h + 2 * pad, W2 = w + 2 * pad;
    const long long total = planes * H2 * W2;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long pl = i / ((long long)H2 * W2);
        const int rem = (int)(i - pl * H2 * W2), y = rem / W2 - pad, x = rem % W2 - pad;
        dst[i] = (y >= 0 && y < h && x >= 0 && x < w) ? __ldg(src + (pl * h + y) * w + x) : 0.f;
    }
}

// wf[c][c'][p][q] = w[c'][c][r-1-p][r-1-q]
__global__ void flip_transpose_kernel(const float *__restrict__ w, float *__restrict__ wf, int Cout, int C, int r) {
    const long long total = (long long)Cout * C * r * r;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int q = (int)(i % r), p = (int)((i / r) % r);
        const long long cc = i / ((long long)r * r);
        const int co = (int)(cc % Cout), c = (int)(cc / Cout);
        wf[i] = __ldg(w + (((long long)co * C + c) * r + (r - 1 - p)) * r + (r - 1 - q));
    }
}

// dst[b][a][k] = src[a][b][k], k < inner
__global__ void swap01_kernel(const float *__restrict__ src, float *__restrict__ dst, int A, int B, long long inner) {
    const long long total = (long long)A * B * inner;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long k = i % inner, ba = i / inner;
        const int a = (int)(ba % A), b = (int)(ba / A);
        dst[i] = __ldg(src + ((long long)a * B + b) * inner + k);
    }
}

unsigned grid_for(long long total) {
    long long g = (total + 255) / 256;
    return (unsigned)(g > 148LL * 32 ? 148LL * 32 : (g < 1 ? 1 : g));
}

}  // namespace

cudaError_t fc_launch_pad(const float *src, float *dst, long long planes, int h, int w, int pad, cudaStream_t s) {
    pad_kernel<<<grid_for(planes * (h + 2 * pad) * (w + 2 * pad)), 256, 0, s>>>(src, dst, planes, h, w, pad);
    return cudaGetLastError();
}

cudaError_t fc_launch_flip_transpose(const float *w, float *wf, int Cout, int C, int r, cudaStream_t s) {
    flip_transpose_kernel<<<grid_for((long long)Cout * C * r * r), 256, 0, s>>>(w, wf, Cout, C, r);
    return cudaGetLastError();
}

cudaError_t fc_launch_swap01(const float *src, float *dst, int A, int B, long long inner, cudaStream_t s) {
    swap01_kernel<<<grid_for((long long)A * B * inner), 256, 0, s>>>(src, dst, A, B, inner);
    return cudaGetLastError();
}
