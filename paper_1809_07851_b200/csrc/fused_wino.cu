// NK2 + NK3 + NK4 fused into one tcgen05 kernel for Winograd F(2x2, 3x3) (SURVEY.md 8(f)
// row 2: the input transform in the contraction's producer, the inverse transform in its
// epilogue; PAPER.md P:455-460 / P:483-486 hand U and X between stages through memory,
// this kernel keeps them on chip).  Option conv_plan_options.fused.
//
// Why only F(2,3), and why N = 16: all E = t^2 products of a tile meet in one epilogue, so
// tensor memory (512 fp32 columns x 128 lanes) must hold E accumulators of N output
// channels; with the transformed input U also resident in TMEM as the MMA's A operand (a
// 4-stage ring of 64 columns) that leaves 256 columns: E N = 16 x 16.  A CTA owns 128 tiles
// x 16 output channels and recomputes its tiles' input transform once per 16-channel block
// of C' (C'/16 times in all): it pays only when C' is small.  (With U in shared memory
// instead -- N = 32, every M128 x N32 x K8 MMA re-reading a 4 KB A tile -- the kernel was
// shared-memory-bound: 2.4-3.8 ms on VGG-1.2 / VGG-3.2.)
//
// One persistent CTA per SM (672 threads, ~151 KB shared memory, all 512 TMEM columns):
//   warp 0       V producer: TMA (32-byte swizzle) of NK1's V_hi / V_lo [z][c'][k] boxes
//                of (8 k, 16 c', 16 z): all elements of one 8-channel K slot per stage
//   warp 1       TMEM allocator; warps 1, 18-20: one MMA-issuing thread per element of the
//                stage, 3 kind::tf32 MMAs each (M 128 tiles, N 16 c', K 8, A from TMEM):
//                U_lo V_hi + U V_lo + U V_hi
//   warps 2-5    input loaders: 8-byte (even W) or 4-byte cp.async, lanes along a row, of the
//                tile block's (2 TBH + 2) x (2 TBW + 2) input patch, 8 channels per slot,
//                zero-filled outside the image (rows are not 16-byte aligned in general: no TMA)
//   warps 6-13   transform: thread (tile = TMEM lane, 4 channels); T = B^T d once per
//                8-channel slot, then per stage the row g of U = T B (elements 4g .. 4g+3)
//                as U (the MMA reads it truncated to TF32) and U_lo = U - trunc_tf32(U),
//                tcgen05.st into the stage's A columns
//   warps 14-17  epilogue: tcgen05.ld of the 16 accumulators of a tile (lane = tile),
//                Y = A^T M A, streaming stores of the 2 x 2 outputs per channel
// Barriers: in_full (cp.async arrivals) / in_empty, a_full (transform warps) / a_empty (MMA
// commit), v_full (TMA) / v_empty (MMA commit), tmem_full (commit) / tmem_empty (epilogue).
#include <cuda.h>

#include "common.h"
#include "winograd_tables.h"
#include "xform_util.cuh"

namespace {

using namespace fcx;

constexpr int FW_THREADS = 672;
constexpr int NCO = 16;   // output channels per CTA (MMA N)
constexpr int BKC = 8;    // channels per K step (tf32 MMA K; one 32-byte swizzle row of V)
constexpr int EG = 4;     // elements per stage (one row of U)
#ifndef FC_FUSED_STAGES
#define FC_FUSED_STAGES 4
#endif
constexpr int STAGES = FC_FUSED_STAGES;  // A (U) ring in TMEM
constexpr int VSTAGES = 6;    // V ring in shared memory, one 8-channel K slot (all 16 elements) per stage
constexpr int IN_SLOTS = 4;
constexpr int ACC_COLS = 16 * NCO;                          // 256: element e at columns e N ..
constexpr int A_COLS = EG * 2 * BKC;                        // 64 per stage: [element][hi, lo][k]
constexpr int B_PLANE = NCO * BKC * 4;                      // 512 bytes: one element of V_hi or V_lo
constexpr int STAGE_BYTES = 2 * 16 * B_PLANE;               // 16384: V_hi [16 el], V_lo [16 el]
constexpr int IN_FLOATS = BKC * 10 * 66;                    // largest patch: TBW = 32 (10 x 66)
constexpr int IN_BYTES = IN_FLOATS * 4;                     // 21120
constexpr int NBAR = 2 * IN_SLOTS + 2 * STAGES + 2 * VSTAGES + 2;
constexpr int SMEM_BYTES = 1024 + VSTAGES * STAGE_BYTES + IN_SLOTS * IN_BYTES + 8 * NBAR + 16;
static_assert(ACC_COLS + STAGES * A_COLS <= 512, "tensor memory columns");
static_assert(SMEM_BYTES <= 232448, "shared memory per CTA");

struct FwArgs {
    const float *in;
    float *out;
    int B, C, Cout, H, W, Ho, Wo, n_h, n_w;
    int lw;                 // log2 of the tile block width TBW (3, 4, 5); TBH = 128 / TBW
    int nbh, nbw, ncb;      // tile blocks per column / row, output-channel blocks of NCO
    int ntasks, nk;         // tasks (image, block row, block column, channel block); K slots
};

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// tcgen05 shared-memory descriptor, K-major with the 32-byte swizzle (layout 6): 8-row
// groups 256 bytes apart
__device__ __forceinline__ uint64_t desc_sw32(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;               // leading byte offset 16 (unused inside one swizzle row)
    d |= (uint64_t)(256 >> 4) << 32;      // stride byte offset
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)6 << 61;
    return d;
}

// D[tmem] (+)= A[tmem] . B[smem]^T, kind::tf32
__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c0, int c1,
                                            int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            dst),
        "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, float a, float b, float c, float d) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(__float_as_uint(a)),
                 "r"(__float_as_uint(b)), "r"(__float_as_uint(c)), "r"(__float_as_uint(d))
                 : "memory");
}

#define TMEM_LD_X4(taddr, v)                                                                          \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"                     \
                 : "=r"((v)[0]), "=r"((v)[1]), "=r"((v)[2]), "=r"((v)[3])                             \
                 : "r"(taddr))

// mbarrier wait for warps off the critical path (epilogue between tasks, loaders and the V
// producer running ahead): back off with nanosleep between probes -- spinning warps' probes
// otherwise crowd the pipe every mbarrier operation of the CTA goes through (ncu: the
// synchronisation probes were 46% of the kernel's instructions)
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity, unsigned ns) {
    uint32_t done;
    for (;;) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
        if (done) return;
        __nanosleep(ns);
    }
}

#ifdef FC_FUSED_TRACE
// debug timeline of CTA 0: [role][event] clock64 stamps (role 0 loader warp 2 slot arrivals,
// 1 transform warp 6 stage arrivals, 2 MMA issuer (warp 1) stage commits, 3 V producer, 4 epilogue)
__device__ long long g_fw_trace[5][1024];
#define FW_TRACE(role, idx)                                                            \
    do {                                                                               \
        if (blockIdx.x == 0 && (idx) < 1024) g_fw_trace[role][idx] = clock64();        \
    } while (0)
#else
#define FW_TRACE(role, idx) \
    do {                    \
    } while (0)
#endif

struct Task {
    int b, ti0, tj0, co0;
};
__device__ __forceinline__ Task decode(const FwArgs &a, int T) {
    Task k;
    const int cb = T % a.ncb;
    int rest = T / a.ncb;
    const int bw = rest % a.nbw;
    rest /= a.nbw;
    const int bh = rest % a.nbh;
    k.b = rest / a.nbh;
    k.ti0 = bh << (7 - a.lw);
    k.tj0 = bw << a.lw;
    k.co0 = cb * NCO;
    return k;
}

// Input loader warp wl: for every task and 8-channel slot, channels 2 wl and 2 wl + 1 of the
// tile block's PH x PW input patch into the slot, lanes along a row (coalesced).  W2: rows are
// 8-byte aligned (W even, x0 even): one 8-byte cp.async per lane per 2 floats.  Copies outside
// the image zero-fill (src-size 0) from a valid address.  (Measured pace: ~5.2 K cycles per
// slot on VGG-1.2 -- the kernel's limit together with the MMA issue rate, DESIGN.md section 11;
// loading through registers instead, 36 coalesced loads per lane, was 2.5x slower.)
template <bool W2, class FullF, class EmptyF>
__device__ __forceinline__ void load_patches(const FwArgs &a, int wl, int lane, uint32_t in0, FullF in_full,
                                             EmptyF in_empty, int PH, int PW) {
    constexpr int VW = W2 ? 2 : 1;  // floats per copy
    int nev = 0;
    (void)nev;
    const int cpr = PW / VW;         // copies per patch row (PW is even)
    int slot = 0;
    uint32_t ph = 0;
    for (int T = blockIdx.x; T < a.ntasks; T += gridDim.x) {
        const Task tk = decode(a, T);
        const int y0 = 2 * tk.ti0, x0 = 2 * tk.tj0;
        int xo[3], nb[3];
        bool act[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const int k = lane + 32 * j, x = x0 + VW * k;
            act[j] = k < cpr;
            nb[j] = x < a.W ? 4 * VW : 0;
            xo[j] = x < a.W ? x : 0;
        }
        for (int kc = 0; kc < a.nk; ++kc) {
            mbar_wait_sleep(in_empty(slot), ph ^ 1, 128);
            const uint32_t dst0 = in0 + slot * IN_BYTES;
#pragma unroll 1
            for (int cc = 0; cc < 2; ++cc) {
                const int c = 2 * wl + cc, ch = kc * BKC + c;
                const bool chok = ch < a.C;
                const float *plane = a.in + ((size_t)tk.b * a.C + (chok ? ch : 0)) * a.H * (size_t)a.W;
                const float *rp = plane + (size_t)y0 * a.W;
                uint32_t d = dst0 + (uint32_t)(c * PH * PW + VW * lane) * 4u;
                const int rows = chok ? min(PH, a.H - y0) : 0;  // rows with data; the rest zero-fill
#pragma unroll 4
                for (int py = 0; py < PH; ++py) {
                    const bool rok = py < rows;
                    const float *rs = rok ? rp : plane;
#pragma unroll
                    for (int j = 0; j < 3; ++j)
                        if (act[j]) {
                            const float *src = rs + xo[j];
                            const int n = rok ? nb[j] : 0;
                            const uint32_t dj = d + 128u * VW * j;
                            if (W2)
                                asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dj), "l"(src), "r"(n)
                                             : "memory");
                            else
                                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dj), "l"(src), "r"(n)
                                             : "memory");
                        }
                    rp += a.W;
                    d += (uint32_t)PW * 4u;
                }
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(in_full(slot)) : "memory");
            if (wl == 0 && lane == 0) FW_TRACE(0, nev++);
            if (++slot == IN_SLOTS) {
                slot = 0;
                ph ^= 1;
            }
        }
    }
}

__global__ void __launch_bounds__(FW_THREADS, 1)
    nk_fused_wino23(const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmVlo, FwArgs a) {
    constexpr wtab::Tables tb = wtab::make(2, 3);  // F(2,3): B^T [4][4], A^T [2][4] as literals
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_addr(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *gbase = smem_raw + (base - raw);
    const uint32_t in0 = base + VSTAGES * STAGE_BYTES;
    const uint32_t bar0 = in0 + IN_SLOTS * IN_BYTES;
    auto in_full = [&](int s) { return bar0 + 8u * s; };
    auto in_empty = [&](int s) { return bar0 + 8u * (IN_SLOTS + s); };
    auto a_full = [&](int s) { return bar0 + 8u * (2 * IN_SLOTS + s); };
    auto a_empty = [&](int s) { return bar0 + 8u * (2 * IN_SLOTS + STAGES + s); };
    auto v_full = [&](int s) { return bar0 + 8u * (2 * IN_SLOTS + 2 * STAGES + s); };
    auto v_empty = [&](int s) { return bar0 + 8u * (2 * IN_SLOTS + 2 * STAGES + VSTAGES + s); };
    const uint32_t tfull = bar0 + 8u * (2 * IN_SLOTS + 2 * STAGES + 2 * VSTAGES);
    const uint32_t tempty = tfull + 8u;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(gbase + (bar0 - base) + 8 * NBAR);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int TBW = 1 << a.lw, TBH = 128 >> a.lw;
    const int PW = 2 * TBW + 2, PH = 2 * TBH + 2;

    if (threadIdx.x == 0) {
        for (int s = 0; s < IN_SLOTS; ++s) {
            mbar_init(in_full(s), 128);  // one cp.async arrival per loader thread
            mbar_init(in_empty(s), 8);   // one arrival per transform warp
        }
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(a_full(s), 8);
            mbar_init(a_empty(s), EG);  // one commit per MMA issuer
        }
        for (int s = 0; s < VSTAGES; ++s) {
            mbar_init(v_full(s), 1);
            mbar_init(v_empty(s), EG);
        }
        mbar_init(tfull, EG);
        mbar_init(tempty, 4);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmVlo) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- V producer
            int stage = 0, nev = 0;
            (void)nev;
            uint32_t ph = 0;
            for (int T = blockIdx.x; T < a.ntasks; T += gridDim.x) {
                const Task tk = decode(a, T);
                for (int kc = 0; kc < a.nk; ++kc) {
                    mbar_wait_sleep(v_empty(stage), ph ^ 1, 64);
                    const uint32_t sb = base + stage * STAGE_BYTES;
                    mbar_expect(v_full(stage), STAGE_BYTES);
                    tma_load_3d(sb, &tmV, v_full(stage), kc * BKC, tk.co0, 0);
                    tma_load_3d(sb + 16 * B_PLANE, &tmVlo, v_full(stage), kc * BKC, tk.co0, 0);
                    FW_TRACE(3, nev++);
                    if (++stage == VSTAGES) {
                        stage = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1 || warp >= 18) {
        if (lane == 0) {  // ---- MMA issuers: warp 1 -> element 4g, warps 18-20 -> 4g + 1 .. 4g + 3
            // (one issuing thread sustains one MMA per ~51 cycles at N <= 64 whatever the shape,
            // tools/probes/mma_small_n.cu; four issuers reach ~15 cycles per M128 x N16 MMA)
            const int j = warp == 1 ? 0 : warp - 17;
            // kind::tf32, D f32, A (TMEM) and B K-major, N = 16, M = 128
            constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NCO >> 3) << 17) |
                                       ((uint32_t)(128 >> 4) << 24);
            const uint64_t bdesc0 = desc_sw32(base);
            int stage = 0, vs = 0, nev = 0;
            uint32_t ph = 0, vph = 0, tph = 0;
            (void)nev;
            for (int T = blockIdx.x; T < a.ntasks; T += gridDim.x) {
                mbar_wait_parity(tempty, tph ^ 1);
                tc_fence_after();
                for (int kc = 0; kc < a.nk; ++kc)
                    for (int g = 0; g < 4; ++g) {
                        mbar_wait_parity(a_full(stage), ph);
                        if (g == 0) mbar_wait_parity(v_full(vs), vph);
                        tc_fence_after();
                        const uint32_t d = tmem_base + (uint32_t)((4 * g + j) * NCO);
                        const uint32_t a_hi = tmem_base + (uint32_t)(ACC_COLS + stage * A_COLS + 2 * j * BKC);
                        const uint32_t a_lo = a_hi + BKC;
                        // descriptor start addresses advance in 16-byte units (stage, plane offsets)
                        const int e = 4 * g + j;
                        const uint64_t b_hi = bdesc0 + (uint64_t)((vs * STAGE_BYTES + e * B_PLANE) >> 4);
                        const uint64_t b_lo = bdesc0 + (uint64_t)((vs * STAGE_BYTES + (16 + e) * B_PLANE) >> 4);
                        mma_tf32_ts(d, a_lo, b_hi, idesc, kc > 0 ? 1u : 0u);
                        mma_tf32_ts(d, a_hi, b_lo, idesc, 1u);
                        mma_tf32_ts(d, a_hi, b_hi, idesc, 1u);
                        mma_commit(a_empty(stage));
                        if (j == 0) FW_TRACE(2, nev++);
                        if (++stage == STAGES) {
                            stage = 0;
                            ph ^= 1;
                        }
                        if (g == 3) {
                            mma_commit(v_empty(vs));
                            if (++vs == VSTAGES) {
                                vs = 0;
                                vph ^= 1;
                            }
                        }
                    }
                mma_commit(tfull);
                tph ^= 1;
            }
        }
    } else if (warp < 6) {  // ---- input loaders: warp wl copies channels 2 wl, 2 wl + 1 of a slot
        if ((a.W & 1) == 0)
            load_patches<true>(a, warp - 2, lane, in0, in_full, in_empty, PH, PW);
        else
            load_patches<false>(a, warp - 2, lane, in0, in_full, in_empty, PH, PW);
    } else if (warp < 14) {  // ---- transform (256 threads: tile = TMEM lane, channels 4q .. 4q+3)
        const int quarter = warp & 3, q = (warp - 6) >> 2;
        const int r = 32 * quarter + lane;
        const int ti = r >> a.lw, tj = r & (TBW - 1);
        const uint32_t tlane = tmem_base + ((uint32_t)(32 * quarter) << 16) + (uint32_t)(ACC_COLS + 4 * q);
        int slot = 0, stage = 0, nev = 0;
        uint32_t iph = 0, ph = 0;
        (void)nev;
        for (int T = blockIdx.x; T < a.ntasks; T += gridDim.x) {
            for (int kc = 0; kc < a.nk; ++kc) {
                mbar_wait_parity(in_full(slot), iph);
                // T[c][k][b] = sum_a B^T[k][a] d[a][b] for the thread's 4 channels
                float Tm[4][4][4];
                const float *ps = reinterpret_cast<const float *>(gbase + (in0 - base) + slot * IN_BYTES) +
                                  (4 * q) * PH * PW + (2 * ti) * PW + 2 * tj;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    float d[4][4];
#pragma unroll
                    for (int y = 0; y < 4; ++y) {
                        const float2 v0 = *reinterpret_cast<const float2 *>(ps + (c * PH + y) * PW);
                        const float2 v1 = *reinterpret_cast<const float2 *>(ps + (c * PH + y) * PW + 2);
                        d[y][0] = v0.x;
                        d[y][1] = v0.y;
                        d[y][2] = v1.x;
                        d[y][3] = v1.y;
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k)
#pragma unroll
                        for (int x = 0; x < 4; ++x) {
                            float s = -0.f;
#pragma unroll
                            for (int y = 0; y < 4; ++y) s = wtab::cfma(tb.BT[k][y], d[y][x], s);
                            Tm[c][k][x] = s;
                        }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive1(in_empty(slot));
                if (++slot == IN_SLOTS) {
                    slot = 0;
                    iph ^= 1;
                }
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    mbar_wait_parity(a_empty(stage), ph ^ 1);
                    tc_fence_after();
                    const uint32_t ts = tlane + (uint32_t)(stage * A_COLS);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        float v[4], lo[4];
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            float s = -0.f;
#pragma unroll
                            for (int x = 0; x < 4; ++x) s = wtab::cfma(tb.BT[j][x], Tm[c][g][x], s);
                            v[c] = s;
                            // U_hi = U (read truncated to TF32 by the MMA), U_lo = U - trunc_tf32(U),
                            // exact in fp32; the MMA truncates U_lo too (2^-21 of |U| per product)
                            lo[c] = s - __uint_as_float(__float_as_uint(s) & 0xFFFFE000u);
                        }
                        tmem_st4(ts + (uint32_t)(2 * j * BKC), v[0], v[1], v[2], v[3]);
                        tmem_st4(ts + (uint32_t)((2 * j + 1) * BKC), lo[0], lo[1], lo[2], lo[3]);
                    }
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive1(a_full(stage));
                    if (warp == 6 && lane == 0) FW_TRACE(1, nev++);
                    if (++stage == STAGES) {
                        stage = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else {  // ---- epilogue (warps 14-17: TMEM lanes 32 (warp % 4) ..)
        const int qd = warp & 3;
        const int r = qd * 32 + lane;
        const int til = r >> a.lw, tjl = r & (TBW - 1);
        const bool v2 = (a.Wo & 1) == 0 && ((reinterpret_cast<uintptr_t>(a.out) & 7) == 0);
        uint32_t tph = 0;
        int nev = 0;
        (void)nev;
        for (int T = blockIdx.x; T < a.ntasks; T += gridDim.x) {
            const Task tk = decode(a, T);
            const int ti = tk.ti0 + til, tj = tk.tj0 + tjl;
            const bool tile_ok = ti < a.n_h && tj < a.n_w;
            const int y = 2 * ti, x = 2 * tj;
            mbar_wait_sleep(tfull, tph, 512);
            if (warp == 14 && lane == 0) FW_TRACE(4, nev++);
            tc_fence_after();
#pragma unroll 1
            for (int cg = 0; cg < NCO / 4; ++cg) {
                uint32_t v[16][4];
                const uint32_t taddr = tmem_base + ((uint32_t)(qd * 32) << 16) + (uint32_t)(cg * 4);
#pragma unroll
                for (int e = 0; e < 16; ++e) TMEM_LD_X4(taddr + (uint32_t)(e * NCO), v[e]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (cg == NCO / 4 - 1) {  // every accumulator read: the next task's MMAs may start
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive1(tempty);
                }
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int co = tk.co0 + cg * 4 + c;
                    // Y = A^T M A: Z[i][b] = sum_j M[i][j] A^T[b][j], Y[a][b] = sum_i A^T[a][i] Z[i][b]
                    float Z[4][2];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int bb = 0; bb < 2; ++bb) {
                            float s = -0.f;
#pragma unroll
                            for (int j = 0; j < 4; ++j) s = wtab::cfma(tb.AT[bb][j], __uint_as_float(v[4 * i + j][c]), s);
                            Z[i][bb] = s;
                        }
                    if (!tile_ok || co >= a.Cout) continue;
                    float *orow = a.out + (((size_t)tk.b * a.Cout + co) * a.Ho + y) * a.Wo + x;
#pragma unroll
                    for (int aa = 0; aa < 2; ++aa) {
                        float o[2];
#pragma unroll
                        for (int bb = 0; bb < 2; ++bb) {
                            float s = -0.f;
#pragma unroll
                            for (int i = 0; i < 4; ++i) s = wtab::cfma(tb.AT[aa][i], Z[i][bb], s);
                            o[bb] = s;
                        }
                        if (y + aa >= a.Ho) continue;
                        float *p = orow + (size_t)aa * a.Wo;
                        if (v2 && x + 1 < a.Wo) {
                            __stcs(reinterpret_cast<float2 *>(p), make_float2(o[0], o[1]));
                        } else {
                            __stcs(p, o[0]);
                            if (x + 1 < a.Wo) __stcs(p + 1, o[1]);
                        }
                    }
                }
            }
            tph ^= 1;
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    }
}

}  // namespace

bool fc_fused_wino23_eligible(const Geometry &g) {
    return g.nd == 0 && g.method == CONV_WINOGRAD && g.m == 2 && g.r == 3 && !g.vf16 && !g.cplx;
}

// Tile block width: the TBW in {8, 16, 32} (TBH = 128 / TBW) with the fewest padded tiles
// (ties: 16); e.g. 28 x 28 tiles (VGG-3.2) -> 4 x 32 blocks, 112 x 112 (VGG-1.2) -> 8 x 16.
int fc_fused_wino23_lw(int n_h, int n_w) {
    int best = 4;
    long long best_cost = -1;
    for (int lw : {4, 3, 5}) {
        const int tbw = 1 << lw, tbh = 128 >> lw;
        const long long cost = (long long)((n_h + tbh - 1) / tbh) * tbh * (long long)((n_w + tbw - 1) / tbw) * tbw;
        if (best_cost < 0 || cost < best_cost) {
            best_cost = cost;
            best = lw;
        }
    }
    return best;
}

cudaError_t fc_launch_fused_wino23(const Geometry &g, const float *in, const float *Vhi, const float *Vlo,
                                   float *out, cudaStream_t s) {
    if (!fc_fused_wino23_eligible(g) || !Vlo) return cudaErrorInvalidValue;
    // V[z][c'][Kp] (NK1's 3xTF32 planes): dims (C, C', 16); reads past C or C' are zero-filled
    const unsigned long long Kp = (unsigned long long)g.Kp;
    const unsigned long long dims[3] = {(unsigned long long)g.C, (unsigned long long)g.Cout, 16ull};
    const unsigned long long strides[2] = {Kp * 4ull, (unsigned long long)g.M * Kp * 4ull};
    const unsigned int box[3] = {BKC, NCO, 16};
    CUtensorMap mV, mVlo;
    if (!fc_tma_encode_f32(&mV, Vhi, 3, dims, strides, box, 32) ||
        !fc_tma_encode_f32(&mVlo, Vlo, 3, dims, strides, box, 32))
        return cudaErrorInvalidValue;
    FwArgs a;
    a.in = in;
    a.out = out;
    a.B = g.B; a.C = g.C; a.Cout = g.Cout; a.H = g.H; a.W = g.W; a.Ho = g.Ho; a.Wo = g.Wo;
    a.n_h = g.n_h; a.n_w = g.n_w;
    a.lw = fc_fused_wino23_lw(g.n_h, g.n_w);
    const int tbw = 1 << a.lw, tbh = 128 >> a.lw;
    a.nbh = (g.n_h + tbh - 1) / tbh;
    a.nbw = (g.n_w + tbw - 1) / tbw;
    a.ncb = (g.Cout + NCO - 1) / NCO;
    const long long ntasks = (long long)g.B * a.nbh * a.nbw * a.ncb;
    if (ntasks >= (1LL << 31)) return cudaErrorInvalidValue;
    a.ntasks = (int)ntasks;
    a.nk = (g.C + BKC - 1) / BKC;
    const void *kern = (const void *)nk_fused_wino23;
    cudaError_t e = fc_smem_attr(kern, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    const int nsm = fc_num_sms();
    const int grid = a.ntasks < nsm ? a.ntasks : nsm;
    nk_fused_wino23<<<grid, FW_THREADS, SMEM_BYTES, s>>>(mV, mVlo, a);
    return cudaGetLastError();
}

#ifdef FC_FUSED_TRACE
extern "C" int fc_fused_trace(long long *host) {
    return (int)cudaMemcpyFromSymbol(host, g_fw_trace, sizeof(long long) * 5 * 1024);
}
#endif
