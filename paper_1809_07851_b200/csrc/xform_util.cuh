// Device helpers shared by the transform translation units (product path only).
#pragma once

#include <stdint.h>

#include "common.h"

// FFT tile edges t with compile-time NK1 / NK2 / NK4 codelets (mixed-radix products of
// 2, 3, 5, 7 and the primes 13 and 31 up to 32; "arbitrary sizes").
#define FC_FFT_TILES(X)                                                                                    \
    X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(12) X(13) X(14) X(15) X(16) X(18) X(20) X(21) X(24) X(25) X(27) \
        X(28) X(30) X(31) X(32)
// (t, m) Winograd pairs with compile-time matrices
#define FC_WINO_TILES(X) X(4, 2) X(4, 3) X(5, 3) X(6, 4) X(6, 2) X(8, 6)


namespace fcx {

// q = a / d for small non-negative integers (a < 2^20, 1 <= d < 2^12) from a float reciprocal:
// (a + 0.5) / d lies at least 0.5 / d away from an integer, far more than the rounding error,
// so the truncation is exact -- 3 instructions instead of a ~20-instruction integer division.
__device__ __forceinline__ int fc_sdiv(int a, float inv_d) { return (int)(((float)a + 0.5f) * inv_d); }

// Copy `rows` staged output rows (pitch SWo floats in smem) to `rows` contiguous rows
// of Wo floats in global memory: one warp per row, lanes along the row (coalesced,
// streaming stores, no per-element division).
__device__ __forceinline__ void store_strip(float *__restrict__ dst, const float *__restrict__ src, int rows, int Wo,
                                            int SWo) {
    if (SWo == Wo && ((((uintptr_t)dst) | ((uintptr_t)src)) & 15) == 0 && (Wo & 3) == 0) {
        // the staged rows have the output's pitch: one flat run of 16-byte vectors
        const float4 *s4 = reinterpret_cast<const float4 *>(src);
        float4 *d4 = reinterpret_cast<float4 *>(dst);
        for (int i = threadIdx.x; i < (rows * Wo) >> 2; i += blockDim.x) __stcs(d4 + i, s4[i]);
        return;
    }
    if ((Wo & 3) == 0 && (SWo & 3) == 0 && ((((uintptr_t)dst) | ((uintptr_t)src)) & 15) == 0) {
        // padded staging pitch (a multiple of 4 floats): 16-byte vectors, flat index over
        // (row, vector) with one float-reciprocal division each (the per-row scalar loop was
        // 19% of the t = 27 FFT NK4's instructions, ncu r02f)
        const int w4 = Wo >> 2, p4 = SWo >> 2;
        const float inv = 1.f / (float)w4;
        const float4 *s4 = reinterpret_cast<const float4 *>(src);
        float4 *d4 = reinterpret_cast<float4 *>(dst);
        for (int i = threadIdx.x; i < rows * w4; i += blockDim.x) {
            const int r = fc_sdiv(i, inv);
            __stcs(d4 + i, s4[r * p4 + (i - r * w4)]);
        }
        return;
    }
    if (SWo == Wo) {  // same pitch, unaligned: one flat scalar run
        for (int i = threadIdx.x; i < rows * Wo; i += blockDim.x) __stcs(dst + i, src[i]);
        return;
    }
    if (Wo < 48) {  // narrow rows: flat index keeps every lane busy; the row from a float
        // reciprocal (fc_sdiv, 3 instructions; the integer division it replaces made the deep
        // layer's Winograd NK4 instruction-bound, ncu r02i)
        const float inv = 1.f / (float)Wo;
        for (int idx = threadIdx.x; idx < rows * Wo; idx += blockDim.x) {
            const int r = fc_sdiv(idx, inv), c = idx - r * Wo;
            __stcs(dst + idx, src[r * SWo + c]);
        }
        return;
    }
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int r = threadIdx.x >> 5; r < rows; r += nw) {
        const float *sr = src + (size_t)r * SWo;
        float *dr = dst + (size_t)r * Wo;
        for (int c = lane; c < Wo; c += 32) __stcs(dr + c, sr[c]);
    }
}

// ------------------------------------------------- TMA bulk-copy helpers ---
// (A TMA plane-pipeline Winograd NK2 / NK4 -- whole image planes streamed into a 3-slot
// shared-memory ring with cp.async.bulk -- measured slower than the thread-per-tile kernels
// on VGG-3.2 F(4,3), NK2 178 vs 150 us, NK4 145 vs 133 us, and was removed in round 2.)

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_init1(uint32_t bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITP_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITP_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}


__device__ __forceinline__ void mbar_arrive1(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// TMA tile loads (no multicast) completing on an mbarrier; coordinates innermost first
__device__ __forceinline__ void tma_load_5d(uint32_t dst, const void *tmap, uint32_t bar, int c0, int c1, int c2,
                                            int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
        "%6}], [%7];" ::"r"(dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const void *tmap, uint32_t bar, int c0, int c1, int c2,
                                            int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5}], [%6];" ::"r"(dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
}
// named barrier `id` over `nthreads` threads (whole warps)
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

}  // namespace fcx
