// NK3 on the 5th-generation tensor cores: the element-wise stage as Z batched
// real products (Eq. 8 "multiplication of a matrix U_e of
// size BN x C with a matrix V_e of size C x C'")
//
//     X_z [M x BN] = V_z [M x K] . U_z [K x BN]        z < Z
//
// computed in fp32 semantics with a 3xTF32 split (reading R11):
//     V.U ~= V_lo.U_hi + V_hi.U_lo + V_hi.U_hi      (fp32 TMEM accumulation),
// V_hi = rna_tf32(V), V_lo = V - V_hi pre-split by NK1 (V is small); the MMA
// reads U truncated to TF32 (measured, dbg/mma_test.cu), so U_hi = U and four
// "splitter" warps write U_lo = U - trunc_tf32(U) next to the TMA-loaded U tile:
// U is read from HBM exactly once per tile and never stored twice.
//
// One persistent, warp-specialised kernel, CG = 1 (one CTA, M = 128) or CG = 2
// (a CTA pair / cluster of 2 issuing cta_group::2 MMAs with M = 256: rank r
// holds V rows [128 r, 128 r + 128) and U columns [r N/2, (r+1) N/2); each
// CTA's TMEM receives its 128 rows x N columns):
//   warp 0      TMA producer: V_hi, V_lo (K-major, 64B/128B swizzle) and U
//               (MN-major, SWIZZLE_128B_ATOM_32B -- the only MN-major swizzle
//               tcgen05 accepts for 32-bit operands) into a STAGES-deep ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (leader CTA)
//   warps 4-7   epilogue: tcgen05.ld 32x32b -> 128B-swizzled smem tile ->
//               TMA bulk tensor store of X (full lines, clipped at M / BN)
//   warps 8-11  splitter: U_lo, fence.proxy.async, one arrival per warp
// mbarriers: full (TMA tx), split (splitters of all CG CTAs -> leader),
// empty and tmem_full (MMA commit, multicast to the pair), tmem_empty
// (epilogue warps of all CG CTAs -> leader).  Cross-CTA arrivals use the
// default .release.cta semantics (as CUTLASS's ClusterBarrier): an explicit
// .release.cluster compiles to a GPU-scope MEMBAR per arrival.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>

#include <cuda_fp16.h>

#include "common.h"

namespace {

__device__ __forceinline__ float rna_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

constexpr int NUM_THREADS = 384;
// F16X3 kernel: warps 0-7 as the tf32 kernel's, then F16_SPLIT_WARPS splitter warps
#ifndef FC_F16_SPLIT_WARPS
#define FC_F16_SPLIT_WARPS 4
#endif
constexpr int F16_SPLIT_WARPS = FC_F16_SPLIT_WARPS;
constexpr int F16_THREADS = 256 + 32 * F16_SPLIT_WARPS;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c0, int c1,
                                            int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            dst),
        "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c0, int c1,
                                            int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
            dst),
        "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// shared-memory matrix descriptor (tcgen05 "version 1"); layout 2 = SWIZZLE_128B,
// 4 = SWIZZLE_64B (K-major operands), 1 = SWIZZLE_128B_BASE32B (MN-major 32-bit)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                              uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}

template <int CG>
struct Tc;  // cta_group-specific instructions

template <>
struct Tc<1> {
    static __device__ __forceinline__ void alloc(uint32_t slot, uint32_t cols) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot), "r"(cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    static __device__ __forceinline__ void dealloc(uint32_t taddr, uint32_t cols) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols));
    }
    static __device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
            "l"(a), "l"(b), "r"(idesc), "r"(acc)
            : "memory");
    }
    static __device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
            "l"(a), "l"(b), "r"(idesc), "r"(acc)
            : "memory");
    }
    static __device__ __forceinline__ void commit(uint32_t bar) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                     : "memory");
    }
    static __device__ __forceinline__ void arrive_leader(uint32_t bar) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
    }
    static __device__ __forceinline__ void sync_all() { __syncthreads(); }
};

template <>
struct Tc<2> {
    static __device__ __forceinline__ void alloc(uint32_t slot, uint32_t cols) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot), "r"(cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    static __device__ __forceinline__ void dealloc(uint32_t taddr, uint32_t cols) {
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols));
    }
    static __device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
            "l"(a), "l"(b), "r"(idesc), "r"(acc)
            : "memory");
    }
    static __device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
            "l"(a), "l"(b), "r"(idesc), "r"(acc)
            : "memory");
    }
    static __device__ __forceinline__ void commit(uint32_t bar) {  // multicast to both CTAs of the pair
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], "
            "%1;" ::"r"(bar),
            "h"((uint16_t)3)
            : "memory");
    }
    static __device__ __forceinline__ void arrive_leader(uint32_t bar) {
        asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(map_to_rank(bar, 0)) : "memory");
    }
    static __device__ __forceinline__ void sync_all() {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
};

#define TMEM_LD_32(taddr, v)                                                                                      \
    asm volatile(                                                                                                 \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                            \
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),        \
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),  \
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),             \
          "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),             \
          "=r"(v[30]), "=r"(v[31])                                                                                \
        : "r"(taddr))

// X stores of an element-sharded contraction (conv_eshard_forward_b_peer): the 32-column box
// at column `col` of the local column space goes to the owner of that column -- peer k's
// receive buffer, through its own tensor map (maps / col: device arrays of n entries, col[k] =
// first column of peer k's segment); n == 0: the plan's own X (tmX).  The exchange is then
// part of the contraction's epilogue: no local X, no pack copies.
struct PeerX {
    const CUtensorMap *maps;
    const long long *col;
    int n;
};
__device__ __forceinline__ void store_x_box(const CUtensorMap *tmX, const PeerX &px, uint32_t sb, int col, int row,
                                            int z) {
    const CUtensorMap *m = tmX;
    int c0 = col;
    if (px.n) {
        int k = 0;
        while (k + 1 < px.n && col >= px.col[k + 1]) ++k;
        m = px.maps + k;
        c0 = col - (int)px.col[k];
    }
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(m), "r"(sb),
                 "r"(c0), "r"(row), "r"(z)
                 : "memory");
}

template <int CG, int BLOCK_N, int STAGES, int BK>
struct TcCfg {
    static constexpr int BM = 128 * CG;       // MMA M (rows of V per tile)
    static constexpr int NH = BLOCK_N / CG;   // columns of U held per CTA
    static constexpr int A_BYTES = 128 * BK * 4;
    static constexpr int B_BYTES = NH * BK * 4;
    static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;  // A_hi, A_lo, B, B_lo
    static constexpr int TX_BYTES = 2 * A_BYTES + B_BYTES;         // bytes TMA lands per stage
    static constexpr int TMEM_COLS = 2 * BLOCK_N;                  // double-buffered accumulator
    static constexpr int EPI_BYTES = 4 * 2 * 32 * 32 * 4;          // per epilogue warp: 2 x (32 rows x 128 B)
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 256;
};

template <int CG, int BLOCK_N, int STAGES, int BK>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    nk3_gemm_tcgen05(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmAlo,
                     const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmX, int M,
                     int K, long long NP, int Z, int cplx, int Mh, int kb_half, PeerX px) {
    using Cfg = TcCfg<CG, BLOCK_N, STAGES, BK>;
    using I = Tc<CG>;
    static_assert(BK == 16 || BK == 32, "BK is one 64 B or 128 B swizzle row");
    static_assert(Cfg::TMEM_COLS <= 512, "TMEM holds 512 columns");
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *gbase = smem_raw + (base - raw);
    const uint32_t epi0 = base + STAGES * Cfg::STAGE_BYTES;  // epilogue staging (1024-aligned)
    const uint32_t bar0 = epi0 + Cfg::EPI_BYTES;
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto split_bar = [&](int s) { return bar0 + 8u * (STAGES + s); };
    auto empty_bar = [&](int s) { return bar0 + 8u * (2 * STAGES + s); };
    auto tfull_bar = [&](int a) { return bar0 + 8u * (3 * STAGES + a); };
    auto tempty_bar = [&](int a) { return bar0 + 8u * (3 * STAGES + 2 + a); };
    uint32_t *tmem_slot =
        reinterpret_cast<uint32_t *>(gbase + STAGES * Cfg::STAGE_BYTES + Cfg::EPI_BYTES + 8 * (3 * STAGES + 4));

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = CG == 2 ? cluster_rank() : 0u;
    const int grp = blockIdx.x / CG, ngrp = gridDim.x / CG;
    const int n_m = (M + Cfg::BM - 1) / Cfg::BM;
    const int n_n = (int)((NP + BLOCK_N - 1) / BLOCK_N);
    const int num_tiles = Z * n_m * n_n;
    const int num_k = (K + BK - 1) / BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(split_bar(s), 4 * CG);  // one arrival per splitter warp of every CTA in the group
            mbar_init(empty_bar(s), 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull_bar(a), 1);
            mbar_init(tempty_bar(a), 4 * CG);  // one arrival per epilogue warp of every CTA in the group
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmAlo) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
    }
    if (warp == 1) I::alloc(smem_u32(tmem_slot), Cfg::TMEM_COLS);
    tc_fence_before();
    I::sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    auto decode = [&](int T, int &z, int &m0, int &n0) {
        const int mb = T % n_m, rest = T / n_m;
        m0 = mb * Cfg::BM;
        n0 = (rest % n_n) * BLOCK_N;
        z = rest / n_n;
    };

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer (every CTA loads its rows of V and columns of U)
            int stage = 0;
            uint32_t phase = 0;
            for (int T = grp; T < num_tiles; T += ngrp) {
                int z, m0, n0;
                decode(T, z, m0, n0);
                for (int kb = 0; kb < num_k; ++kb) {
                    mbar_wait(empty_bar(stage), phase ^ 1);
                    const uint32_t sA = base + stage * Cfg::STAGE_BYTES;
                    const uint32_t sAlo = sA + Cfg::A_BYTES;
                    const uint32_t sB = sA + 2 * Cfg::A_BYTES;
                    mbar_expect_tx(full_bar(stage), Cfg::TX_BYTES);
                    int ak = kb * BK, ar = m0 + 128 * (int)rank, az = z;
                    if (cplx) {  // Re rows: [V_r | -V_i], Im rows: [V_i | V_r] over K = [U_r; U_i]
                        const int re = m0 < Mh, hi = kb >= kb_half;
                        ak = (kb - hi * kb_half) * BK;
                        ar -= re ? 0 : Mh;
                        az = 2 * z + (re ? hi : 1 - hi);
                    }
                    tma_load_3d(sA, &tmA, full_bar(stage), ak, ar, az);
                    tma_load_3d(sAlo, &tmAlo, full_bar(stage), ak, ar, az);
#pragma unroll
                    for (int j = 0; j < Cfg::NH / 32; ++j) {  // U blocked by FC_TB tiles: (t, z, k, block)
                        const int nc = n0 + (int)rank * Cfg::NH + 32 * j;
                        tma_load_4d(sB + j * (BK * 128), &tmB, full_bar(stage), nc % FC_TB, z, kb * BK, nc / FC_TB);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {  // ---- MMA issuer (leader CTA)
            // kind::tf32, D f32, A K-major, B MN-major, M = 128*CG, N = BLOCK_N
            const uint32_t idesc0 = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (1u << 16) |
                                    ((uint32_t)(BLOCK_N >> 3) << 17) | ((uint32_t)(Cfg::BM >> 4) << 24);
            constexpr uint32_t a_sbo = BK * 4 * 8, a_layout = BK == 32 ? 2u : 4u;
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int T = grp; T < num_tiles; T += ngrp) {
                mbar_wait(tempty_bar(acc), acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BLOCK_N;
                const bool re_tile = cplx && (T % n_m) * Cfg::BM < Mh;
                for (int kb = 0; kb < num_k; ++kb) {
                    mbar_wait(split_bar(stage), phase);
                    tc_fence_after();
                    // complex mode: the Re rows' second K half multiplies -V_i (A negate bit)
                    const uint32_t idesc = (re_tile && kb >= kb_half) ? (idesc0 | (1u << 13)) : idesc0;
                    const uint32_t sA = base + stage * Cfg::STAGE_BYTES;
                    const uint32_t sAlo = sA + Cfg::A_BYTES;
                    const uint32_t sB = sA + 2 * Cfg::A_BYTES;
                    const uint32_t sBlo = sB + Cfg::B_BYTES;
#pragma unroll
                    for (int s = 0; s < BK / 8; ++s) {
                        // A: +32 B per K=8 step inside the swizzled row; B: +1024 B = 8 K-rows
                        const uint64_t a_hi = make_desc(sA + 32 * s, 16, a_sbo, a_layout);
                        const uint64_t a_lo = make_desc(sAlo + 32 * s, 16, a_sbo, a_layout);
                        const uint64_t b_hi = make_desc(sB + 1024 * s, BK * 128, 512, 1);
                        const uint64_t b_lo = make_desc(sBlo + 1024 * s, BK * 128, 512, 1);
                        const uint32_t first = (kb == 0 && s == 0) ? 0u : 1u;
                        I::mma(d_tmem, a_lo, b_hi, idesc, first);
                        I::mma(d_tmem, a_hi, b_lo, idesc, 1u);
                        I::mma(d_tmem, a_hi, b_hi, idesc, 1u);
                    }
                    I::commit(empty_bar(stage));
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                I::commit(tfull_bar(acc));
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ---- epilogue: each warp drains its 32 TMEM lanes, 32 columns at a time, into a
        // 128B-swizzled 32 x 32 smem tile and TMA-stores it (full lines, clipped at M / NP).
        const int q = warp & 3;
        const uint32_t stage0 = epi0 + q * (2 * 4096);
        int acc = 0, buf = 0;
        uint32_t acc_phase = 0;
        for (int T = grp; T < num_tiles; T += ngrp) {
            int z, m0, n0;
            decode(T, z, m0, n0);
            mbar_wait(tfull_bar(acc), acc_phase);
            tc_fence_after();
            const int row0 = m0 + 128 * (int)rank + q * 32;
#pragma unroll 1
            for (int c = 0; c < BLOCK_N / 32; ++c) {
                uint32_t v[32];
                const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BLOCK_N + c * 32;
                TMEM_LD_32(taddr, v);
                // the staging buffer about to be overwritten must have been read by its TMA store
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                __syncwarp();
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                const uint32_t sb = stage0 + buf * 4096;
                const uint32_t rowaddr = sb + lane * 128;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rowaddr + ((j ^ (lane & 7)) << 4)),
                                 "r"(v[4 * j]), "r"(v[4 * j + 1]), "r"(v[4 * j + 2]), "r"(v[4 * j + 3])
                                 : "memory");
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    store_x_box(&tmX, px, sb, n0 + 32 * c, row0, z);
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
                buf ^= 1;
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) I::arrive_leader(tempty_bar(acc));
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    } else if (warp >= 8) {  // ---- splitter: lo = U - trunc_tf32(U)
        const int st = threadIdx.x - 256;
        int stage = 0;
        uint32_t phase = 0;
        for (int T = grp; T < num_tiles; T += ngrp) {
            for (int kb = 0; kb < num_k; ++kb) {
                mbar_wait(full_bar(stage), phase);
                const float4 *bh =
                    reinterpret_cast<const float4 *>(gbase + stage * Cfg::STAGE_BYTES + 2 * Cfg::A_BYTES);
                float4 *bl = reinterpret_cast<float4 *>(gbase + stage * Cfg::STAGE_BYTES + 2 * Cfg::A_BYTES +
                                                        Cfg::B_BYTES);
#pragma unroll
                for (int j = 0; j < Cfg::B_BYTES / 16 / 128; ++j) {
                    const float4 v = bh[st + 128 * j];
                    // U_hi = trunc_tf32(U) is what the MMA reads from the staged U; U_lo = U - U_hi
                    // is exact in fp32 and rounded to the nearest TF32 here (the MMA would
                    // truncate it: 2^-21 instead of 2^-22 relative to |U|)
                    float4 lo;
                    lo.x = rna_tf32(v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u));
                    lo.y = rna_tf32(v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u));
                    lo.z = rna_tf32(v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u));
                    lo.w = rna_tf32(v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u));
                    bl[st + 128 * j] = lo;
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if ((st & 31) == 0) I::arrive_leader(split_bar(stage));
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    }

    tc_fence_before();
    I::sync_all();
    if (warp == 1) {
        tc_fence_after();
        I::dealloc(tmem_base, Cfg::TMEM_COLS);
    }
}

// ---------------------------------------------------------------------------
// F16X3 variant (conv_gemm_impl CONV_GEMM_TCGEN05_F16X3, reading R16):
// tcgen05.mma kind::f16 (fp16 x fp16 -> fp32, twice the kind::tf32 rate) on
// scaled two-term fp16 splits, three products per K step as above:
//     s_v s_u (V.U) ~= V'_lo.U'_hi + V'_hi.U'_lo + V'_hi.U'_hi
// V' = s_v[c'] V pre-split by NK1 into fp16 (V'_hi, V'_lo) planes, K-major,
// TMA-loaded with the 64 B swizzle (32 K per row); U arrives as fp32 (NK2's
// output, read from HBM once per tile) and the four splitter warps write
// U'_hi = rn_f16(s_u U), U'_lo = rn_f16(s_u U - U'_hi) K-major in the same
// 64 B-swizzled layout (row = tile column n, 16-byte chunk = 8 K values).
// s_u = s_u[b] = 2^(15 - e) with max|U_b| < 2^e over image b's tiles (NK2's per-image
// reduction), so |s_u U| < 2^15 and no fp16 overflows, and an image's arithmetic does
// not depend on the rest of its batch; the epilogue multiplies accumulator (c', n) by
// 1 / (s_u[b(n)] s_v[c']) (exact powers of two) before the TMA store of X.
template <int CG, int BLOCK_N, int SA, int SU, bool GC = false>
struct TcCfgF16 {
    // GC (Gauss epilogue combine): the three products T1, T2, T3 of one (e, c', n) tile
    // go to three of four TMEM accumulator slots, the epilogue stores Re = T1 - T3 and
    // Im = T1 + T2 (two staging boxes per chunk); otherwise a double-buffered accumulator
    static constexpr int NACC = GC ? 4 : 2;
    static constexpr int SUB = GC ? 3 : 1;         // accumulators (products) per output tile
    static constexpr int BK = 32;              // K per stage (one 64 B swizzle row of fp16)
    static constexpr int BM = 128 * CG;
    static constexpr int NH = BLOCK_N / CG;    // tile columns (n) held per CTA
    static constexpr int A_BYTES = 128 * BK * 2;
    static constexpr int UF_BYTES = NH * BK * 4;   // fp32 U as TMA lands it: [BK][NH]
    static constexpr int B_BYTES = NH * BK * 2;    // one fp16 split plane: [NH][BK] swizzled
    static constexpr int A_STAGE = 2 * A_BYTES + 2 * B_BYTES;  // MMA operands: V'_hi, V'_lo, U'_hi, U'_lo
    static constexpr int TMEM_COLS = NACC * BLOCK_N;
    static constexpr int EPI_BYTES = 4 * (GC ? 4 : 2) * 32 * 32 * 4;
    static constexpr int NBARS = 3 * SA + 2 * SU + 2 * NACC;
    static constexpr int SMEM_BYTES = SA * A_STAGE + SU * UF_BYTES + EPI_BYTES + 1024 + 8 * NBARS + 16;
};

__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
    const __half2 h = __floats2half2_rn(a, b);  // .x = a (low half), .y = b
    return *reinterpret_cast<const uint32_t *>(&h);
}

// Two rings: the MMA-operand ring (SA stages: V' via TMA, U' written by the
// splitters) and a deeper fp32 U staging ring (SU stages) that the splitters
// release as soon as they have converted a stage -- so the U loads from HBM run
// SU stages ahead of the tensor cores instead of waiting for MMA completion.
// Warp 0 lane 0 streams U, warp 2 lane 0 streams V (independent run-ahead).
template <int CG, int BLOCK_N, int SA, int SU, bool GC>
__global__ void __launch_bounds__(F16_THREADS, 1)
    nk3_gemm_tcgen05_f16(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmAlo,
                         const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmX, int M,
                         int K, long long NP, int Z, int cplx, int Mh, int kb_half, int Cout,
                         const unsigned int *__restrict__ umax_p, const float *__restrict__ inv_sv, FastDiv divN,
                         int BNr, PeerX px) {
    using Cfg = TcCfgF16<CG, BLOCK_N, SA, SU, GC>;
    using I = Tc<CG>;
    constexpr int BK = Cfg::BK, NACC = Cfg::NACC, SUB = Cfg::SUB;
    static_assert(Cfg::TMEM_COLS <= 512, "TMEM holds 512 columns");
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *gbase = smem_raw + (base - raw);
    const uint32_t ubase = base + SA * Cfg::A_STAGE;           // fp32 U ring
    const uint32_t epi0 = ubase + SU * Cfg::UF_BYTES;
    const uint32_t bar0 = epi0 + Cfg::EPI_BYTES;
    auto fullA_bar = [&](int s) { return bar0 + 8u * s; };                 // V landed (tx)
    auto split_bar = [&](int s) { return bar0 + 8u * (SA + s); };          // U' written (4 CG warps)
    auto emptyA_bar = [&](int s) { return bar0 + 8u * (2 * SA + s); };     // MMA done (commit)
    auto fullU_bar = [&](int s) { return bar0 + 8u * (3 * SA + s); };      // fp32 U landed (tx)
    auto emptyU_bar = [&](int s) { return bar0 + 8u * (3 * SA + SU + s); };  // converted (4 local warps)
    auto tfull_bar = [&](int a) { return bar0 + 8u * (3 * SA + 2 * SU + a); };
    auto tempty_bar = [&](int a) { return bar0 + 8u * (3 * SA + 2 * SU + NACC + a); };
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(gbase + (bar0 - base) + 8 * Cfg::NBARS);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = CG == 2 ? cluster_rank() : 0u;
    const int grp = blockIdx.x / CG, ngrp = gridDim.x / CG;
    const int n_m = (M + Cfg::BM - 1) / Cfg::BM;
    const int n_n = (int)((NP + BLOCK_N - 1) / BLOCK_N);
    // GC: Z = 3E products; an output tile (unit) is the element e's three sub-tiles z = e + p E
    const int Zu = GC ? Z / 3 : Z;
    const int num_tiles = Zu * n_m * n_n;
    const int num_k = (K + BK - 1) / BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < SA; ++s) {
            mbar_init(fullA_bar(s), 1);
            mbar_init(split_bar(s), F16_SPLIT_WARPS * CG);
            mbar_init(emptyA_bar(s), 1);
        }
        for (int s = 0; s < SU; ++s) {
            mbar_init(fullU_bar(s), 1);
            mbar_init(emptyU_bar(s), F16_SPLIT_WARPS);
        }
        for (int a = 0; a < NACC; ++a) {
            mbar_init(tfull_bar(a), 1);
            mbar_init(tempty_bar(a), 4 * CG);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmAlo) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmU) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
    }
    if (warp == 1) I::alloc(smem_u32(tmem_slot), Cfg::TMEM_COLS);
    tc_fence_before();
    I::sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    auto decode = [&](int T, int &z, int &m0, int &n0) {
        const int mb = T % n_m, rest = T / n_m;
        m0 = mb * Cfg::BM;
        n0 = (rest % n_n) * BLOCK_N;
        z = rest / n_n;
    };
    // per-image U scale s_u[b] = 2^(15 - e), max|U_b| < 2^e (NK2's per-image reduction);
    // column n < BNr belongs to image n / N (padding columns: image 0, their X is never read)
    auto col_scale = [&](int col) {
        return fc_pow2_scale(__uint_as_float(umax_p[col < BNr ? fc_div(col, divN) : 0]), 15);
    };

    if (warp == 0) {
        if (lane == 0) {  // ---- U producer: fp32 U columns of this CTA into the staging ring
            int su = 0;
            uint32_t pu = 0;
            for (int T = grp; T < num_tiles; T += ngrp) {
                int z0, m0, n0;
                decode(T, z0, m0, n0);
                for (int p = 0; p < SUB; ++p)
                for (int kb = 0; kb < num_k; ++kb) {
                    const int z = z0 + p * Zu;
                    mbar_wait(emptyU_bar(su), pu ^ 1);
                    mbar_expect_tx(fullU_bar(su), Cfg::UF_BYTES);
                    {  // U blocked by FC_TB tiles: box (NH tiles, 1, BK, 1) of block (n0 + rank NH) / FC_TB
                        const int nc = n0 + (int)rank * Cfg::NH;
                        tma_load_4d(ubase + su * Cfg::UF_BYTES, &tmU, fullU_bar(su), nc % FC_TB, z, kb * BK,
                                    nc / FC_TB);
                    }
                    if (++su == SU) {
                        su = 0;
                        pu ^= 1;
                    }
                }
            }
        }
    } else if (warp == 2) {
        if (lane == 0) {  // ---- V producer: V'_hi, V'_lo (fp16) rows of this CTA
            int sa = 0;
            uint32_t pa = 0;
            for (int T = grp; T < num_tiles; T += ngrp) {
                int z0, m0, n0;
                decode(T, z0, m0, n0);
                for (int p = 0; p < SUB; ++p)
                for (int kb = 0; kb < num_k; ++kb) {
                    const int z = z0 + p * Zu;
                    mbar_wait(emptyA_bar(sa), pa ^ 1);
                    const uint32_t sA = base + sa * Cfg::A_STAGE;
                    mbar_expect_tx(fullA_bar(sa), 2 * Cfg::A_BYTES);
                    int ak = kb * BK, ar = m0 + 128 * (int)rank, az = z;
                    if (cplx) {
                        const int re = m0 < Mh, hi = kb >= kb_half;
                        ak = (kb - hi * kb_half) * BK;
                        ar -= re ? 0 : Mh;
                        az = 2 * z + (re ? hi : 1 - hi);
                    }
                    tma_load_3d(sA, &tmA, fullA_bar(sa), ak, ar, az);
                    tma_load_3d(sA + Cfg::A_BYTES, &tmAlo, fullA_bar(sa), ak, ar, az);
                    if (++sa == SA) {
                        sa = 0;
                        pa ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {  // ---- MMA issuer (leader CTA)
            // kind::f16: D f32 (bit 4), A = B = f16 (0), both K-major, N >> 3 at 17, M >> 4 at 24
            const uint32_t idesc0 = (1u << 4) | ((uint32_t)(BLOCK_N >> 3) << 17) | ((uint32_t)(Cfg::BM >> 4) << 24);
            const uint64_t desc0 = make_desc(base, 16, 512, 4);
            int sa = 0;
            uint32_t pa = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int T = grp; T < num_tiles; T += ngrp)
            for (int p = 0; p < SUB; ++p) {
                mbar_wait(tempty_bar(acc), acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BLOCK_N;
                const bool re_tile = cplx && (T % n_m) * Cfg::BM < Mh;
                for (int kb = 0; kb < num_k; ++kb) {
                    mbar_wait(split_bar(sa), pa);
                    tc_fence_after();
                    const uint32_t idesc = (re_tile && kb >= kb_half) ? (idesc0 | (1u << 13)) : idesc0;
                    // descriptors = the stage-0 A_hi descriptor + (byte offset >> 4): the start
                    // address is the descriptor's low field, so one add each (the single issuing
                    // thread's per-MMA work bounds narrow tiles)
                    const uint64_t dst = desc0 + (uint64_t)((uint32_t)(sa * Cfg::A_STAGE) >> 4);
#pragma unroll
                    for (int s = 0; s < BK / 16; ++s) {  // K = 16 per instruction: +32 B in the 64 B row
                        const uint64_t a_hi = dst + 2 * s;
                        const uint64_t a_lo = dst + (Cfg::A_BYTES >> 4) + 2 * s;
                        const uint64_t b_hi = dst + ((2 * Cfg::A_BYTES) >> 4) + 2 * s;
                        const uint64_t b_lo = dst + ((2 * Cfg::A_BYTES + Cfg::B_BYTES) >> 4) + 2 * s;
                        const uint32_t first = (kb == 0 && s == 0) ? 0u : 1u;
                        I::mma_f16(d_tmem, a_lo, b_hi, idesc, first);
                        I::mma_f16(d_tmem, a_hi, b_lo, idesc, 1u);
                        I::mma_f16(d_tmem, a_hi, b_hi, idesc, 1u);
                    }
                    I::commit(emptyA_bar(sa));
                    if (++sa == SA) {
                        sa = 0;
                        pa ^= 1;
                    }
                }
                I::commit(tfull_bar(acc));
                if (++acc == NACC) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (GC && warp >= 4 && warp < 8) {
        // ---- Gauss epilogue combine: Re = T1 - T3 -> X rows c', Im = T1 + T2 -> rows C' + c'
        // of plane e; unscaled as above; two 32 x 32 boxes per chunk
        const int q = warp & 3;
        const uint32_t stage0 = epi0 + q * (4 * 4096);
        int acc = 0, buf = 0;
        uint32_t acc_phase = 0;
        for (int T = grp; T < num_tiles; T += ngrp) {
            int e, m0, n0;
            decode(T, e, m0, n0);
            const int row0 = m0 + 128 * (int)rank + q * 32;
            const int cp = row0 + lane;
            const float rs = cp < Cout ? __ldg(inv_sv + cp) : 0.f;
            int a[3];
#pragma unroll
            for (int p = 0; p < 3; ++p) {  // the three slots of this tile, in issue order
                a[p] = acc;
                mbar_wait(tfull_bar(acc), acc_phase);
                if (++acc == NACC) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
            tc_fence_after();
            const bool live = row0 < Cout;  // C' % 32 == 0: a box is all-valid or all-outside
#pragma unroll 1
            for (int c = 0; c < BLOCK_N / 32; ++c) {
                uint32_t v1[32], v2[32], v3[32];
                const float inv_col = 1.f / col_scale(n0 + 32 * c + lane);  // lane = column here
                const uint32_t tl = tmem_base + ((uint32_t)(q * 32) << 16) + c * 32;
                TMEM_LD_32(tl + a[0] * BLOCK_N, v1);
                TMEM_LD_32(tl + a[1] * BLOCK_N, v2);
                TMEM_LD_32(tl + a[2] * BLOCK_N, v3);
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                __syncwarp();
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                const uint32_t sre = stage0 + buf * 8192, sim = sre + 4096;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    float re[4], im[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const float t1 = __uint_as_float(v1[4 * j + i]);
                        const float sc = rs * __shfl_sync(0xffffffffu, inv_col, 4 * j + i);
                        re[i] = (t1 - __uint_as_float(v3[4 * j + i])) * sc;
                        im[i] = (t1 + __uint_as_float(v2[4 * j + i])) * sc;
                    }
                    const uint32_t o = lane * 128 + ((j ^ (lane & 7)) << 4);
                    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(sre + o), "f"(re[0]), "f"(re[1]),
                                 "f"(re[2]), "f"(re[3])
                                 : "memory");
                    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(sim + o), "f"(im[0]), "f"(im[1]),
                                 "f"(im[2]), "f"(im[3])
                                 : "memory");
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    if (live) {
                        asm volatile(
                            "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                                &tmX),
                            "r"(sre), "r"(n0 + 32 * c), "r"(row0), "r"(e)
                            : "memory");
                        asm volatile(
                            "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                                &tmX),
                            "r"(sim), "r"(n0 + 32 * c), "r"(Cout + row0), "r"(e)
                            : "memory");
                    }
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
                buf ^= 1;
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0)
#pragma unroll
                for (int p = 0; p < 3; ++p) I::arrive_leader(tempty_bar(a[p]));
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    } else if (!GC && warp >= 4 && warp < 8) {
        // ---- epilogue: unscale by 1 / (s_u s_v[c']) and TMA-store X (as the tf32 kernel)
        const int q = warp & 3;
        const uint32_t stage0 = epi0 + q * (2 * 4096);
        int acc = 0, buf = 0;
        uint32_t acc_phase = 0;
        for (int T = grp; T < num_tiles; T += ngrp) {
            int z, m0, n0;
            decode(T, z, m0, n0);
            const int row0 = m0 + 128 * (int)rank + q * 32;
            int cp = row0 + lane;
            cp = cp >= Cout ? cp - Cout : cp;  // rows [C', 2C') of the Regular-FFT products: Im of c'
            const float rs = cp < Cout ? __ldg(inv_sv + cp) : 0.f;
            mbar_wait(tfull_bar(acc), acc_phase);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < BLOCK_N / 32; ++c) {
                uint32_t v[32];
                const float inv_col = 1.f / col_scale(n0 + 32 * c + lane);  // lane = column here
                const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BLOCK_N + c * 32;
                TMEM_LD_32(taddr, v);
                if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                __syncwarp();
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    v[j] = __float_as_uint(__uint_as_float(v[j]) * (rs * __shfl_sync(0xffffffffu, inv_col, j)));
                const uint32_t sb = stage0 + buf * 4096;
                const uint32_t rowaddr = sb + lane * 128;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rowaddr + ((j ^ (lane & 7)) << 4)),
                                 "r"(v[4 * j]), "r"(v[4 * j + 1]), "r"(v[4 * j + 2]), "r"(v[4 * j + 3])
                                 : "memory");
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    store_x_box(&tmX, px, sb, n0 + 32 * c, row0, z);
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
                buf ^= 1;
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) I::arrive_leader(tempty_bar(acc));
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    } else if (warp >= 8) {
        // ---- splitter: fp32 U [BK][NH] -> scaled fp16 (hi, lo), K-major 64 B-swizzled rows
        const int st = threadIdx.x - 256;
        constexpr int NSPL = 32 * F16_SPLIT_WARPS;
        static_assert(NSPL % Cfg::NH == 0, "a splitter thread converts one tile column n = st % NH");
        const int ncol = st % Cfg::NH;
        int sa = 0, su = 0;
        uint32_t pa = 0, pu = 0;
        for (int T = grp; T < num_tiles; T += ngrp) {
        int z0_, m0_, n0_;
        decode(T, z0_, m0_, n0_);
        const float su_scale = col_scale(n0_ + (int)rank * Cfg::NH + ncol);  // this column's image
        for (int p = 0; p < SUB; ++p) {
            for (int kb = 0; kb < num_k; ++kb) {
                mbar_wait(fullU_bar(su), pu);
                // the operand slot is free once the MMAs that read it committed (the V producer waits
                // on the same phase); converting does not wait for this stage's V to land -- only
                // the arrival below does, so the conversion overlaps the V load
                mbar_wait(emptyA_bar(sa), pa ^ 1);
                const float *uf = reinterpret_cast<const float *>(gbase + (ubase - base) + su * Cfg::UF_BYTES);
                uint8_t *bh = gbase + sa * Cfg::A_STAGE + 2 * Cfg::A_BYTES;
                uint8_t *bl = bh + Cfg::B_BYTES;
#pragma unroll
                for (int i = 0; i < Cfg::NH * BK / 8 / NSPL; ++i) {
                    const int chunk = st + NSPL * i;
                    const int n = ncol, kg = chunk / Cfg::NH;  // 8 K values kg*8.. of column n
                    float x[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) x[j] = uf[(kg * 8 + j) * Cfg::NH + n] * su_scale;
                    uint32_t h[4], l[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        h[j] = pack_half2(x[2 * j], x[2 * j + 1]);
                        const __half2 hv = *reinterpret_cast<const __half2 *>(&h[j]);
                        const float2 hf = __half22float2(hv);
                        l[j] = pack_half2(x[2 * j] - hf.x, x[2 * j + 1] - hf.y);
                    }
                    const int off = n * 64 + (((kg ^ (n >> 1)) & 3) << 4);
                    *reinterpret_cast<uint4 *>(bh + off) = make_uint4(h[0], h[1], h[2], h[3]);
                    *reinterpret_cast<uint4 *>(bl + off) = make_uint4(l[0], l[1], l[2], l[3]);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if ((st & 31) == 0) {
                    mbar_wait(fullA_bar(sa), pa);  // this CTA's V landed: the split arrival carries it
                    I::arrive_leader(split_bar(sa));
                    Tc<1>::arrive_leader(emptyU_bar(su));  // local: the staging slot may be refilled
                }
                if (++sa == SA) {
                    sa = 0;
                    pa ^= 1;
                }
                if (++su == SU) {
                    su = 0;
                    pu ^= 1;
                }
            }
        }
        }
    }

    tc_fence_before();
    I::sync_all();
    if (warp == 1) {
        tc_fence_after();
        I::dealloc(tmem_base, Cfg::TMEM_COLS);
    }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

// U blocked by FC_TB tiles: dims (t, z, k, nb) = (FC_TB, Z, K, NP / FC_TB), box (b0, 1, b2, 1)
bool encode_u4d(CUtensorMap *map, const void *ptr, uint64_t Z, uint64_t K, uint64_t NP, uint32_t b0, uint32_t b2,
                CUtensorMapSwizzle swz) {  // U[nb][z][k][t] (fc_u_off)
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[4] = {FC_TB, Z, K, NP / FC_TB};
    cuuint64_t strides[3] = {K * FC_TB * 4, FC_TB * 4, K * Z * FC_TB * 4};  // z, k, nb
    cuuint32_t box[4] = {b0, 1, b2, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void *>(ptr), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool encode_3d(CUtensorMap *map, const void *ptr, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1_bytes,
               uint64_t s2_bytes, uint32_t b0, uint32_t b1, CUtensorMapSwizzle swz,
               CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[3] = {d0, d1, d2};
    cuuint64_t strides[2] = {s1_bytes, s2_bytes};
    cuuint32_t box[3] = {b0, b1, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, dt, 3, const_cast<void *>(ptr), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}


template <int CG, int BLOCK_N, int STAGES, int BK>
cudaError_t launch(const Geometry &g, const float *Vhi, const float *Vlo, const float *U, float *X,
                   cudaStream_t s) {
    using Cfg = TcCfg<CG, BLOCK_N, STAGES, BK>;
    static_assert(Cfg::SMEM_BYTES <= 232448, "shared memory per CTA");
    CUtensorMap mA, mAlo, mB, mX;
    const uint64_t Z = (uint64_t)g.Z, M = (uint64_t)g.M, K = (uint64_t)g.K, NP = (uint64_t)g.BN_pad;
    const uint64_t Kp = (uint64_t)g.Kp;
    const CUtensorMapSwizzle aswz = BK == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    // V: [Z][M][Kp], or in complex mode the (V_r, V_i) planes [E][2][C'][Kp] with K = C
    const uint64_t vK = g.cplx ? (uint64_t)g.C : K, vM = g.cplx ? (uint64_t)g.Cout : M;
    const uint64_t vZ = g.cplx ? 2 * (uint64_t)g.E : Z;
    if (!encode_3d(&mA, Vhi, vK, vM, vZ, Kp * 4, vM * Kp * 4, BK, 128, aswz) ||
        !encode_3d(&mAlo, Vlo, vK, vM, vZ, Kp * 4, vM * Kp * 4, BK, 128, aswz) ||
        !encode_u4d(&mB, U, Z, K, NP, 32, BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) ||
        !encode_3d(&mX, X, NP, M, Z, NP * 4, M * NP * 4, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B))
        return cudaErrorInvalidValue;
    auto kern = nk3_gemm_tcgen05<CG, BLOCK_N, STAGES, BK>;
    {
        cudaError_t e = fc_smem_attr((const void *)kern, Cfg::SMEM_BYTES);
        if (e != cudaSuccess) return e;
    }
    const int g_num_sms = fc_num_sms();
    const long long n_m = (g.M + Cfg::BM - 1) / Cfg::BM;
    const long long n_n = (g.BN_pad + BLOCK_N - 1) / BLOCK_N;
    const long long tiles = (long long)g.Z * n_m * n_n;
    const long long groups = tiles < g_num_sms / CG ? tiles : g_num_sms / CG;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(CG * groups));
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = CG > 1 ? 1 : 0;
    if (CG > 1) {  // persistent: no more clusters than fit at once (else a second wave)
        const int mc = fc_max_clusters((const void *)kern, &cfg);
        if (mc > 0 && groups > mc) cfg.gridDim = dim3((unsigned)(CG * mc));
    }
    int M_ = g.M, K_ = g.K, Z_ = g.Z;
    long long NP_ = g.BN_pad;
    int cplx_ = g.cplx, Mh_ = g.Cout, kbh_ = (g.C + BK - 1) / BK;
    if (g.cplx && (g.Cout % Cfg::BM != 0 || g.C % BK != 0)) return cudaErrorInvalidValue;
    const PeerX px{reinterpret_cast<const CUtensorMap *>(g.peer_maps), g.peer_col, g.npeer};
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, mA, mAlo, mB, mX, M_, K_, NP_, Z_, cplx_, Mh_, kbh_, px);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}


template <int CG, int BLOCK_N, int SA, int SU, bool GC = false>
cudaError_t launch_f16(const Geometry &g, const void *Vhi, const void *Vlo, const float *U, float *X,
                       cudaStream_t s) {
    using Cfg = TcCfgF16<CG, BLOCK_N, SA, SU, GC>;
    static_assert(Cfg::SMEM_BYTES <= 232448, "shared memory per CTA");
    CUtensorMap mA, mAlo, mU, mX;
    const uint64_t Z = (uint64_t)g.Z, M = (uint64_t)g.M, K = (uint64_t)g.K, NP = (uint64_t)g.BN_pad;
    const uint64_t Kp = (uint64_t)g.Kp;  // fp16 elements, multiple of 8
    const uint64_t vK = g.cplx ? (uint64_t)g.C : K, vM = g.cplx ? (uint64_t)g.Cout : M;
    const uint64_t vZ = g.cplx ? 2 * (uint64_t)g.E : Z;
    if (!encode_3d(&mA, Vhi, vK, vM, vZ, Kp * 2, vM * Kp * 2, Cfg::BK, 128, CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_DATA_TYPE_FLOAT16) ||
        !encode_3d(&mAlo, Vlo, vK, vM, vZ, Kp * 2, vM * Kp * 2, Cfg::BK, 128, CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_DATA_TYPE_FLOAT16) ||
        !encode_u4d(&mU, U, Z, K, NP, Cfg::NH, Cfg::BK, CU_TENSOR_MAP_SWIZZLE_NONE) ||
        !encode_3d(&mX, X, NP, (uint64_t)g.Xm, (uint64_t)g.Xz, NP * 4, (uint64_t)g.Xm * NP * 4, 32, 32,
                   CU_TENSOR_MAP_SWIZZLE_128B))
        return cudaErrorInvalidValue;
    if (GC && (g.Z != 3 * g.E || g.Xm != 2 * g.Cout || g.Cout % 32 != 0)) return cudaErrorInvalidValue;
    if (GC && g.npeer) return cudaErrorInvalidValue;  // the combine epilogue stores through tmX only
    auto kern = nk3_gemm_tcgen05_f16<CG, BLOCK_N, SA, SU, GC>;
    {
        cudaError_t e = fc_smem_attr((const void *)kern, Cfg::SMEM_BYTES);
        if (e != cudaSuccess) return e;
    }
    const int g_num_sms = fc_num_sms();
    const long long n_m = (g.M + Cfg::BM - 1) / Cfg::BM;
    const long long n_n = (g.BN_pad + BLOCK_N - 1) / BLOCK_N;
    const long long tiles = (long long)(GC ? g.E : g.Z) * n_m * n_n;
    const long long groups = tiles < g_num_sms / CG ? tiles : g_num_sms / CG;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(CG * groups));
    cfg.blockDim = dim3(F16_THREADS);
    cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = CG > 1 ? 1 : 0;
    if (CG > 1) {  // persistent: no more clusters than fit at once (else a second wave)
        const int mc = fc_max_clusters((const void *)kern, &cfg);
        if (mc > 0 && groups > mc) cfg.gridDim = dim3((unsigned)(CG * mc));
    }
    int M_ = g.M, K_ = g.K, Z_ = g.Z, Cout_ = g.Cout;
    long long NP_ = g.BN_pad;
    int cplx_ = g.cplx, Mh_ = g.Cout, kbh_ = (g.C + Cfg::BK - 1) / Cfg::BK;
    if (g.cplx && (g.Cout % Cfg::BM != 0 || g.C % Cfg::BK != 0)) return cudaErrorInvalidValue;
    const unsigned int *um = g.umax;
    const float *isv = g.vscale + g.Cout;
    if (g.BN >= (1LL << 31)) return cudaErrorInvalidValue;
    const FastDiv dN = g.divN;
    const int BNr = (int)g.BN;
    cudaError_t e =
        cudaLaunchKernelEx(&cfg, kern, mA, mAlo, mU, mX, M_, K_, NP_, Z_, cplx_, Mh_, kbh_, Cout_, um, isv, dN, BNr,
                           PeerX{reinterpret_cast<const CUtensorMap *>(g.peer_maps), g.peer_col, g.npeer});
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace

int fc_tcgen05_available() { return get_encode() != nullptr; }

bool fc_tma_encode_f32(void *map, const void *ptr, int rank, const unsigned long long *dims,
                       const unsigned long long *strides_bytes, const unsigned int *box, int swizzle_bytes) {
    auto enc = get_encode();
    if (!enc || rank < 1 || rank > 5) return false;
    CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_NONE;
    if (swizzle_bytes == 32) swz = CU_TENSOR_MAP_SWIZZLE_32B;
    else if (swizzle_bytes == 64) swz = CU_TENSOR_MAP_SWIZZLE_64B;
    else if (swizzle_bytes == 128) swz = CU_TENSOR_MAP_SWIZZLE_128B;
    else if (swizzle_bytes != 0) return false;
    cuuint64_t d[5], st[4];
    cuuint32_t bx[5], es[5];
    for (int i = 0; i < rank; ++i) {
        d[i] = dims[i];
        bx[i] = box[i];
        es[i] = 1;
        if (i + 1 < rank) st[i] = strides_bytes[i];
    }
    CUresult r = enc(reinterpret_cast<CUtensorMap *>(map), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)rank,
                     const_cast<void *>(ptr), d, st, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

cudaError_t fc_launch_gemm_tcgen05(const Geometry &g, const float *Vhi, const float *Vlo, const float *U, float *X,
                                   cudaStream_t s) {
    if (!Vlo) return cudaErrorInvalidValue;
    const int force_1cta = g.tc_1sm;
    // M > 128: CTA pairs (M = 256 per MMA); M <= 128: single CTAs (M = 128 per MMA)
    if (g.M > 128 && !force_1cta) return launch<2, 256, 6, 16>(g, Vhi, Vlo, U, X, s);
    return launch<1, 256, 4, 16>(g, Vhi, Vlo, U, X, s);
}

cudaError_t fc_launch_gemm_tcgen05_f16(const Geometry &g, const void *Vhi, const void *Vlo, const float *U, float *X,
                                       cudaStream_t s) {
    if (!Vlo || !g.umax || !g.vscale) return cudaErrorInvalidValue;
    const int force_1cta = g.tc_1sm;
    // rings (operand stages, fp32 U stages): 4/4 measured 163 us vs 3/6 170 us on VGG-3.2 F(4,3)
    if (g.gc) {  // Gauss epilogue combine: 4 accumulator slots of 128 columns
        if (g.M > 128 && !force_1cta) return launch_f16<2, 128, 5, 4, true>(g, Vhi, Vlo, U, X, s);
        return launch_f16<1, 128, 3, 3, true>(g, Vhi, Vlo, U, X, s);
    }
    // N = 256 tiles unless that pads B N by >= 25% more than N = 128 tiles would (small
    // batches of few-tile images: deep FFT m = 14 has B N = 64, 4x / 2x padded)
    const long long n256 = (g.BN + 255) / 256 * 256, n128 = (g.BN + 127) / 128 * 128;
    if (g.M > 128 && !force_1cta && 4 * n256 >= 5 * n128) return launch_f16<2, 128, 5, 4>(g, Vhi, Vlo, U, X, s);
    if (g.M > 128 && !force_1cta) return launch_f16<2, 256, 4, 4>(g, Vhi, Vlo, U, X, s);
    return launch_f16<1, 128, 4, 4>(g, Vhi, Vlo, U, X, s);
}
