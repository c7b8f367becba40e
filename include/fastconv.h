/*
 * fastconv.h -- C-ABI of the B200-native tiled fast-convolution forward pass.
 *
 * Problem statement (Eq. 5 "eq:forward"): one ConvNet
 * layer's forward propagation
 *
 *     out[b][c'][i][j] = sum_{c<C} sum_{p<r} sum_{q<r} in[b][c][i+p][j+q] * w[c'][c][p][q]
 *
 * (valid cross-correlation, stride 1, no bias; readings R1-R3), for
 * 0 <= i < H-r+1, 0 <= j < W-r+1, computed by one of
 *
 *   CONV_WINOGRAD     Winograd F(m^2, r^2)          (Eq. 1, Eq. 4)
 *   CONV_REGULAR_FFT  Regular-FFT F(m^2, r^2)       (Eq. 2, "Regular-FFT")
 *   CONV_GAUSS_FFT    Gauss-FFT G(m^2, r^2)         (Gauss' 3-mult product)
 *   CONV_DIRECT       direct check path             (north_star step (4))
 *
 * in the paper's four stages: kernel transform (NK1), input
 * transform over overlapping t = m+r-1 tiles (NK2), element-wise
 * stage as E batched matrix products X_e = U_e V_e (NK3), and
 * inverse transform + crop (NK4).  Every stage is a hand-written
 * sm_100a CUDA kernel; the contraction runs on tcgen05 tensor cores with a
 * two-term operand split (F16X3 by default, or 3xTF32; an FFMA fallback is
 * selectable), and Gauss-FFT may be recombined in its epilogue (x_planes).
 *
 * Conventions for every entry point:
 *   - All tensors are fp32, contiguous, row-major: in [B][C][H][W],
 *     w [Cout][C][r][r], out [B][Cout][H-r+1][W-r+1].
 *   - Device pointers must be device memory of the plan's device, 16-byte
 *     aligned (torch allocations are).  The caller owns in/w/out/workspace.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Functions never abort or throw; they return a conv_status.  On error a
 *     thread-local detail string is available from conv_last_error().
 *   - conv_forward is asynchronous on `stream` and performs no host sync.
 *   - A plan is immutable after conv_plan/conv_plan_ex; concurrent forwards on
 *     one plan are safe when their workspace and output buffers are distinct.
 */
#ifndef FASTCONV_H_
#define FASTCONV_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CONV_OK = 0,
    CONV_ERR_INVALID_ARG = 1,     /* bad sizes, NULL pointer, misaligned pointer, short workspace */
    CONV_ERR_UNSUPPORTED = 2,     /* valid but not implemented (e.g. Winograd t > 8, FFT t > 64) */
    CONV_ERR_OUT_OF_MEMORY = 3,   /* plan-constant allocation failed */
    CONV_ERR_CUDA = 4,            /* a CUDA runtime/driver call or launch failed */
    CONV_ERR_DEVICE_MISMATCH = 5  /* pointer or current device differs from the plan's device */
} conv_status;

typedef enum {
    CONV_DIRECT = 0,
    CONV_WINOGRAD = 1,
    CONV_REGULAR_FFT = 2,
    CONV_GAUSS_FFT = 3
} conv_method;

/* Contraction (NK3) implementation.  Both tcgen05 modes hold fp32 accuracy with
 * a two-term split of each operand and three tensor-core products (small terms
 * first), X ~= V_lo U_hi + V_hi U_lo + V_hi U_hi, accumulated in fp32 in TMEM:
 *   3XTF32  kind::tf32; V_hi = rna_tf32(V), V_lo = V - V_hi, U_hi = trunc_tf32(U)
 *           (what the MMA reads), U_lo = U - U_hi.  2^-22-relative products.
 *   F16X3   kind::f16 (2x the tf32 tensor rate): scaled fp16 splits
 *           a_hi = rn_f16(s a), a_lo = rn_f16(s a - a_hi) with exact power-of-two
 *           scales -- one per output channel c' for V (from max|W[c']| times the
 *           transform's norm bound, written by NK1) and one per image b for U
 *           (from max|U_b| reduced by NK2, so an image's result never depends on
 *           the rest of its batch) -- removed again in the epilogue; the
 *           same 22 significant bits as 3xTF32 and no fp16 overflow by construction
 *           (reading R16). */
typedef enum {
    CONV_GEMM_AUTO = 0,            /* tcgen05 F16X3 (the fastest mode that meets the bars) */
    CONV_GEMM_TCGEN05_3XTF32 = 1,  /* tcgen05.mma kind::tf32, TMEM accumulators, hi/lo split */
    CONV_GEMM_FFMA = 2,            /* fp32 FFMA tiled GEMM (the fallback it is measured against) */
    CONV_GEMM_TCGEN05_F16X3 = 3    /* tcgen05.mma kind::f16, scaled fp16 hi/lo split */
} conv_gemm_impl;

typedef struct conv_plan_s *conv_plan_t;

/* Plan options (conv_plan_opts / conv_plan_query_opts).  Every choice a plan makes
 * is a function of (B, C, C', H, W, r, method, m) and these options only -- the
 * library reads no environment variables.  Initialise with conv_plan_options_init()
 * (the defaults are the measured-best settings) and override fields; a NULL options
 * pointer means the defaults.  Invalid values -> CONV_ERR_INVALID_ARG. */
typedef struct {
    int struct_size;          /* sizeof(conv_plan_options), set by conv_plan_options_init */
    conv_gemm_impl gemm;      /* contraction implementation (default CONV_GEMM_AUTO = F16X3) */
    int gauss_combine;        /* Gauss-FFT with F16X3 and C' % 32 == 0: combine Re = T1 - T3,
                                 Im = T1 + T2 in the contraction's epilogue (X at w = 2,
                                 P:427-441).  -1 (default): the stage-sum model decides
                                 (P:772-780); 0: never; 1: whenever eligible */
    int complex_mode;         /* Regular-FFT with tcgen05, C' % 256 == 0, C % 16 (32 for F16X3)
                                 == 0: store V as (V_r, V_i) planes and negate V_i in the MMA.
                                 -1 (default): when eligible; 0: store the real embedding */
    int chunk_images;         /* 0 (default): NK2 -> NK3 -> NK4 over the whole batch; k > 0:
                                 in chunks of k images (L2-resident U / X; measured slower) */
    int generic_transforms;   /* 0 (default): compile-time-t transform kernels where they
                                 exist; 1: always the runtime-t kernels (reference / tests) */
    int single_cta_mma;       /* 0 (default): CTA-pair contraction tiles when M > 128;
                                 1: single-CTA tiles */
    int e2e_chunks;           /* pipelining depth of conv_forward_host (0 = default 8) */
    int overlap_kernel_transform;  /* -1 (default): NK1 runs on a plan-owned stream concurrently
                                 with NK2 (they are independent; NK3 waits for both); 0: serial */
    int fused;                /* Winograd F(2,3) (m = 2, r = 3, 2-D) with the 3xTF32 contraction:
                                 NK2, NK3 and NK4 in ONE tcgen05 kernel -- the input transform in
                                 the contraction's producer, the inverse transform in its epilogue,
                                 U and X never leave the SM (PAPER.md P:455-460,
                                 P:483-486 stream them through memory).  0 (default): staged
                                 kernels; 1: fused (CONV_ERR_UNSUPPORTED unless eligible; gemm
                                 AUTO then resolves to CONV_GEMM_TCGEN05_3XTF32, chunk_images 0).
                                 Pays for small C' (the input transform is recomputed C'/32 times) */
} conv_plan_options;

/* Fill `o` with the defaults (NULL-safe). */
void conv_plan_options_init(conv_plan_options *o);

/* Geometry and algorithmic cost of a plan (PAPER.md
 * Table "layer-stuff" P:1008-1042 with c = C, c' = C', alpha = 1). */
typedef struct {
    int B, C, Cout, H, W, r, m, method;
    int Ho, Wo;
    int t;              /* tile edge m + r - 1 */
    int n_h, n_w;       /* tiles per dimension ceil((H-r+1)/m) */
    int N;              /* tiles per image n_h * n_w */
    int h;              /* stored columns per transformed row: t (Winograd) or t/2+1 (FFT) */
    int E;              /* transformed elements per tile: t*t or t*h */
    int planes;         /* real planes per element: 1 Winograd, 2 Regular (re/im), 3 Gauss */
    long long BN;       /* B * N: rows of U_e / X_e */
    long long BN_pad;   /* BN rounded up to 128 (row pitch of U and X) */
    int gemm_Z, gemm_M, gemm_K;  /* batched contraction: Z products of [M x K] x [K x BN] */
    size_t bytes_U, bytes_V, bytes_X;   /* workspace tensors (V includes the hi/lo split) */
    size_t workspace_bytes;
    /* algorithmic bytes / FLOPs per stage: [0]=NK1 kernel transform,
     * [1]=NK2 input transform, [2]=NK3 contraction, [3]=NK4 output transform */
    double alg_bytes[4];
    double alg_flops[4];
    double direct_flops;  /* 2 B C C' Ho Wo r^2 */
    /* L2-resident batch chunking: conv_forward runs NK1 once, then NK2 -> NK3 -> NK4
     * for `chunk` images at a time, so U and X of a chunk stay in the 126 MB L2 between
     * stages.  bytes_U / bytes_X / BN_pad above are per chunk. */
    int chunk;          /* images per chunk (== B when not chunked) */
    int nchunks;        /* ceil(B / chunk) */
    int gemm;           /* the contraction implementation the plan runs (conv_gemm_impl;
                           CONV_GEMM_AUTO resolved; conv_plan_query reports AUTO's default) */
    /* N-dimensional plans (conv_plan_nd): nd = 1..3 and the per-axis sizes right-aligned in
     * 3 slots (slot 2 = the last, fastest axis; unused leading slots hold 1).  2-D plans report
     * nd = 2 with slots 1, 2 = (H, W); H, W, r, m, t, n_h, n_w above then describe the last
     * two axes. */
    int nd;
    int in_shape[3], kernel_shape[3], m_shape[3], t_shape[3], tiles[3], out_shape[3];
    int x_planes;       /* real planes of X per transformed element: 1 Winograd, 2 Regular-FFT,
                           3 Gauss-FFT (T1, T2, T3), or 2 when the F16X3 contraction combines
                           Gauss in its epilogue (Re = T1 - T3, Im = T1 + T2; C' % 32 == 0;
                           X is then [E][2C'][BN_pad] like Regular-FFT's); 0 for CONV_DIRECT */
    int fused;          /* 1: NK2-NK4 run as one fused kernel (conv_plan_options.fused; no U / X
                           in the workspace, alg_bytes[1] = alg_bytes[3] = 0 and alg_bytes[2] the
                           fused kernel's input + V + output) */
} conv_plan_info;

/* Host-only: validate arguments and fill `info` (no CUDA calls).  m = 0 for a
 * fast method selects the model's tile (conv_plan_best_m).  Errors:
 * INVALID_ARG if any size < 1, H < r, W < r, or m < 0;
 * UNSUPPORTED for Winograd with r < 2, m < 2 or t > 8, or FFT with t > 64.
 * conv_plan_query reports CONV_GEMM_AUTO's plan; conv_plan_query_opts the plan
 * `opts` (NULL = defaults) would build, e.g. for another contraction mode. */
conv_status conv_plan_query(int B, int C, int Cout, int H, int W, int r,
                            conv_method method, int m, conv_plan_info *info);
conv_status conv_plan_query_opts(int B, int C, int Cout, int H, int W, int r,
                                 conv_method method, int m, const conv_plan_options *opts,
                                 conv_plan_info *info);

/* Host-only tile-size planner (the paper's comparison rule
 * "each method at its best m"): for a fast method, evaluate the paper's
 * stage-sum running-time model (per stage max(FLOPs / peak, bytes /
 * bandwidth), summed) with B200 constants -- HBM 6.53 TB/s, the contraction
 * mode's tensor ceiling, and per-kernel-family efficiencies measured on B200
 * -- for every output tile m whose transforms are compiled
 * (Winograd t <= 8; FFT t <= 32), and return the m of least predicted time
 * (ties: the smaller m).  *m_out gets that m, *model_ms its predicted
 * time (may be NULL).  n_cand / cand_m / cand_ms (may be NULL) receive up to
 * max_cand (m, predicted ms) pairs in increasing m.  CONV_DIRECT -> INVALID_ARG. */
conv_status conv_plan_best_m(int B, int C, int Cout, int H, int W, int r, conv_method method,
                             const conv_plan_options *opts, int *m_out, double *model_ms,
                             int max_cand, int *n_cand, int *cand_m, double *cand_ms);
/* The paper's comparison rule across methods (each method at its best m, the fastest
 * wins) on the same model: *method_out / *m_out get the predicted-fastest fast method and its
 * tile, *model_ms (may be NULL) its predicted time.  Errors as conv_plan_best_m. */
conv_status conv_plan_best_method(int B, int C, int Cout, int H, int W, int r, const conv_plan_options *opts,
                                  conv_method *method_out, int *m_out, double *model_ms);

/* Create a plan on the current CUDA device, which must be sm_100 (B200; the library
 * carries sm_100a code only -- other devices get CONV_ERR_UNSUPPORTED) (uploads ~KB of constants:
 * Winograd matrices built exactly in rationals, DFT twiddles computed in fp64,
 * both rounded once to fp32).  m is ignored for CONV_DIRECT; m = 0 for a fast
 * method takes conv_plan_best_m's tile (conv_plan_get_info reports it).  `*out`
 * is set only on CONV_OK; release with conv_destroy.  conv_plan_ex(gemm) is
 * conv_plan_opts with the defaults and that contraction mode. */
conv_status conv_plan(conv_plan_t *out, int B, int C, int Cout, int H, int W, int r,
                      conv_method method, int m);
conv_status conv_plan_ex(conv_plan_t *out, int B, int C, int Cout, int H, int W, int r,
                         conv_method method, int m, conv_gemm_impl gemm);
conv_status conv_plan_opts(conv_plan_t *out, int B, int C, int Cout, int H, int W, int r,
                           conv_method method, int m, const conv_plan_options *opts);

/* N-dimensional and non-isotropic layers ("support an arbitrary
 * number of dimensions, as well as non-isotropic kernels"): nd = 1, 2 or 3 spatial axes,
 *   in  [B][C][in_shape[0]]...[in_shape[nd-1]],   w [C'][C][kernel_shape[0]]...,
 *   out [B][C'][in_shape[d] - kernel_shape[d] + 1 ...]      (valid cross-correlation),
 * with output tile m[d] per axis (t_d = m[d] + kernel_shape[d] - 1; Winograd F(m_d, r_d)
 * per axis with t_d <= 8, r_d = 1 axes are identities; FFT t_d <= 64 with the half
 * spectrum on the last axis).  The transforms are the generic separable kernels of
 * transforms_nd.cu; the contraction is the same tcgen05 / FFMA NK3.  nd = 2 with a square
 * kernel and equal tiles is the 2-D plan (the compile-time codelets).  m is ignored for
 * CONV_DIRECT (may be NULL).  All other entry points (conv_forward, _cached, _host, graphs,
 * timers) accept these plans.  Errors as conv_plan, plus INVALID_ARG for nd outside 1..3 or
 * NULL shape arrays, UNSUPPORTED for tiles whose t-volume exceeds 12800 elements. */
conv_status conv_plan_nd(conv_plan_t *out, int nd, int B, int C, int Cout, const int *in_shape,
                         const int *kernel_shape, conv_method method, const int *m,
                         const conv_plan_options *opts);
conv_status conv_plan_query_nd(int nd, int B, int C, int Cout, const int *in_shape, const int *kernel_shape,
                               conv_method method, const int *m, const conv_plan_options *opts,
                               conv_plan_info *info);

conv_status conv_plan_get_info(conv_plan_t p, conv_plan_info *info);

/* Bytes of device workspace conv_forward needs (U + V + X; 0 for CONV_DIRECT). */
size_t conv_workspace_bytes(conv_plan_t p);

/* Full forward pass, all four stages: NK1 w -> V, NK2 in -> U,
 * NK3 (U, V) -> X, NK4 X -> out.  Asynchronous on `stream`. */
conv_status conv_forward(conv_plan_t p, const float *in, const float *w, float *out,
                         void *workspace, size_t workspace_bytes, void *stream);

/* Same, but synchronises and reports per-stage milliseconds measured with
 * CUDA events: stage_ms[0..3] = NK1, NK2, NK3, NK4 (NK5 for CONV_DIRECT in [2]). */
conv_status conv_forward_profiled(conv_plan_t p, const float *in, const float *w, float *out,
                                  void *workspace, size_t workspace_bytes, void *stream,
                                  float stage_ms[4]);

/* End-to-end call with HOST buffers: copies h_in, h_w (pinned for overlap) to the
 * caller-provided device buffers d_in, d_w, runs the forward pass, copies d_out
 * back to h_out.  The batch is pipelined in image chunks (
 * conv_plan_options.e2e_chunks, default 8): H2D of chunk i+1, the kernels of chunk i and D2H of chunk i-1
 * overlap on plan-owned copy streams.  Asynchronous: when `stream` (the
 * caller's) completes, h_out holds the result (the caller synchronises). */
conv_status conv_forward_host(conv_plan_t p, const float *h_in, const float *h_w, float *h_out,
                              float *d_in, float *d_w, float *d_out,
                              void *workspace, size_t workspace_bytes, void *stream);

/* Inference with cached weight transforms: the kernel
 * transform V depends only on the weights, so conv_transform_weights() runs NK1
 * once into the V region of `workspace`, and every later conv_forward_cached()
 * runs NK2 -> NK3 -> NK4 only, reading that V.  The workspace must keep its V
 * region intact between the calls (U / X are overwritten as usual).  Same
 * results as conv_forward, bit for bit. */
conv_status conv_transform_weights(conv_plan_t p, const float *w, void *workspace, size_t workspace_bytes,
                                   void *stream);
conv_status conv_forward_cached(conv_plan_t p, const float *in, float *out, void *workspace,
                                size_t workspace_bytes, void *stream);

/* Run a single stage (0 = NK1, 1 = NK2, 2 = NK3, 3 = NK4) on the plan's
 * workspace layout for the first chunk (images [0, chunk)); used by stage-level
 * tests.  Arguments a stage does not read may be NULL. */
conv_status conv_run_stage(conv_plan_t p, int stage, const float *in, const float *w, float *out,
                           void *workspace, size_t workspace_bytes, void *stream);

/* Byte offsets of V (hi), V_lo, U and X inside the workspace ([0..3]).  V_hi and
 * V_lo are fp32 (3XTF32 / FFMA) or fp16 (F16X3) [Z][M][Kp] planes. */
conv_status conv_workspace_layout(conv_plan_t p, size_t offsets[4]);
/* F16X3 plans: byte offsets of the per-output-channel scales (fp32 [2][C']:
 * s_v[c'] then 1/s_v[c'], exact powers of two) and of the per-image max|U_b|
 * words (fp32 bits, [chunk] of them) inside the workspace; both 0 for other plans. */
conv_status conv_workspace_aux(conv_plan_t p, size_t offsets[2]);

/* The plan's Winograd matrices in fp64 (exact rationals): AT [m][t], BT [t][t],
 * G [t][r], so that y = AT[(G g) . (BT d)] (Eq. 1).  UNSUPPORTED for
 * non-Winograd plans. */
conv_status conv_plan_winograd_matrices(conv_plan_t p, double *AT, double *BT, double *G);
conv_status conv_winograd_matrices(int m, int r, double *AT, double *BT, double *G);

void conv_destroy(conv_plan_t p);                 /* NULL-safe */
const char *conv_status_string(conv_status s);    /* static string, never NULL */
const char *conv_last_error(void);                /* thread-local detail of the last error */

/* Kernel launches one conv_forward issues for this plan (for gpu_launches):
 * 1 + 3 * nchunks (fast methods; 2 + 3 * nchunks for F16X3 FFT plans, whose kernel
 * transform has a per-c' scale prologue) or 1 (direct).  F16X3 plans also issue one
 * 4-byte memset (the max|U| reset) per chunk. */
int conv_forward_launch_count(conv_plan_t p);

/* Per-stage timing without host synchronisation inside a timed loop:
 * conv_forward_timed() is conv_forward() plus a CUDA event recorded on `stream`
 * before the first and after every kernel launch (events pre-created by
 * conv_timer_create: one call consumes at most launch_count + 2 of the max_launches + 64: a start marker on each stream, NK1 running on the plan's auxiliary stream).  conv_timer_read()
 * synchronises on the last event and returns, per stage, the sum of the recorded
 * launch durations in ms (stage_ms[0..3] = NK1..NK4; the direct path reports in
 * [2]) and the number of launches recorded.  conv_timer_reset() rewinds. */
typedef struct conv_timer_s *conv_timer_t;
conv_status conv_timer_create(conv_timer_t *t, int max_launches);
conv_status conv_forward_timed(conv_plan_t p, const float *in, const float *w, float *out,
                               void *workspace, size_t workspace_bytes, void *stream, conv_timer_t t);
conv_status conv_timer_read(conv_timer_t t, float stage_ms[4], int *launches);
void conv_timer_reset(conv_timer_t t);
void conv_timer_destroy(conv_timer_t t);   /* NULL-safe */

/* CUDA graphs of the forward pass (launch-bound layers, fixed buffers):
 * conv_graph_create() captures `steps` consecutive conv_forward() calls (or, with
 * cached != 0, conv_forward_cached() calls reading the V already in `workspace`)
 * on the given device buffers into one instantiated CUDA graph; conv_graph_launch()
 * replays it asynchronously on `stream` (results identical to the eager calls, bit
 * for bit).  The buffers are baked into the graph: they must stay allocated, and
 * replays read whatever `in` / `w` hold at launch time.  Errors as conv_forward
 * (argument checks happen at creation); `*graph_out` is set only on CONV_OK. */
typedef struct conv_graph_s *conv_graph_t;
conv_status conv_graph_create(conv_plan_t p, const float *in, const float *w, float *out, void *workspace,
                              size_t workspace_bytes, int steps, int cached, conv_graph_t *graph_out);
conv_status conv_graph_launch(conv_graph_t g, void *stream);
void conv_graph_destroy(conv_graph_t g);   /* NULL-safe */

/* Backward passes (not in the paper).  Both gradients of Eq. 5 are
 * valid cross-correlations and run through the same fast pipeline after a re-layout:
 *   which = 1  conv_backward_data:   dx[b][c][y][x] = sum_{c',p,q} dy[b][c'][y-p][x-q] w[c'][c][p][q]
 *              (forward of the (r-1)-zero-padded dy [B][C'][H+r-1][W+r-1] with the flipped,
 *              channel-transposed kernel; method / m as for conv_plan, m = 0: the planner's)
 *   which = 2  conv_backward_filter: dw[c'][c][p][q] = sum_{b,i,j} dy[b][c'][i][j] x[b][c][i+p][j+q]
 *              (forward of x with images and channels swapped against dy as an Ho x Wo kernel:
 *              FFT tiles of the whole image, t = H, W <= 64, or CONV_DIRECT; m is ignored;
 *              Winograd -> UNSUPPORTED)
 * dy [B][C'][H-r+1][W-r+1], w [C'][C][r][r], x / dx [B][C][H][W], dw [C'][C][r][r], all
 * device memory; the workspace holds the re-laid-out operands and the inner forward's
 * U / V / X (conv_workspace_bytes).  Backward plans work only with these two calls. */
conv_status conv_plan_backward(conv_plan_t *out, int which, int B, int C, int Cout, int H, int W, int r,
                               conv_method method, int m, const conv_plan_options *opts);
conv_status conv_backward_data(conv_plan_t p, const float *dy, const float *w, float *dx, void *workspace,
                               size_t workspace_bytes, void *stream);
conv_status conv_backward_filter(conv_plan_t p, const float *x, const float *dy, float *dw, void *workspace,
                                 size_t workspace_bytes, void *stream);

/* Element-sharded multi-GPU execution.  The contraction is E
 * independent products X_e = V_e U_e, so rank j of `world` can own the
 * transformed elements e in [e0_j, e1_j) (an even split of E) for every image while the
 * transforms stay with the images: rank j transforms its batch[j] images (NK2 / NK4) and
 * only its E_j / E share of the kernels (NK1), instead of every rank transforming and
 * reading all of V as the batch-sharded plan does.  One forward is three calls with two
 * all-to-alls (and one tiny all-gather) in between, done by the caller with its
 * communicator (NCCL over NVLink in bench/parallel.py):
 *   conv_eshard_forward_a  NK1 (own elements), NK2 (own images), U packed per peer into
 *                          u_send (peer-major, u_send_bytes[k] to peer k), and this rank's
 *                          per-image max|U_b| (F16X3 scale inputs) into umax_out[batch[rank]]
 *   caller                 all-to-all u_send -> u_recv (u_recv_bytes[k] from peer k);
 *                          all-gather umax_out -> umax_all[sum batch] in rank order
 *   conv_eshard_forward_b  NK3 for own elements over every image's tiles; X packed per peer
 *   caller                 all-to-all x_send -> x_recv
 *   conv_eshard_forward_c  X chunks placed, NK4 for own images -> out[batch[rank]][C'][Ho][Wo]
 * in [batch[rank]][C][H][W] and w [C'][C][r][r] on this rank's device.  Results equal
 * conv_forward of the whole batch bit for bit (same per-column arithmetic).  Buffers are the
 * caller's (device memory of the plan's device); sizes from conv_eshard_sizes (arrays of
 * `world` entries, may be NULL).  NK1 uses the generic kernel (its element range).
 * Errors: INVALID_ARG for bad rank/world/batch, the direct method, or short buffers;
 * UNSUPPORTED when E < world. */
typedef struct conv_eshard_s *conv_eshard_t;
conv_status conv_eshard_create(conv_eshard_t *out, int world, int rank, const int *batch, int C, int Cout, int H,
                               int W, int r, conv_method method, int m, const conv_plan_options *opts);
conv_status conv_eshard_sizes(conv_eshard_t e, size_t *workspace_bytes, size_t *u_send_bytes,
                              size_t *u_recv_bytes, size_t *x_send_bytes, size_t *x_recv_bytes);
conv_status conv_eshard_get_info(conv_eshard_t e, conv_plan_info *local_plan, int *e_lo, int *e_count);
conv_status conv_eshard_forward_a(conv_eshard_t e, const float *in, const float *w, void *u_send, float *umax_out,
                                  void *workspace, size_t workspace_bytes, void *stream);
conv_status conv_eshard_forward_b(conv_eshard_t e, const void *u_recv, const float *umax_all, void *x_send,
                                  void *workspace, size_t workspace_bytes, void *stream);
conv_status conv_eshard_forward_c(conv_eshard_t e, const void *x_recv, float *out, void *workspace,
                                  size_t workspace_bytes, void *stream);
void conv_eshard_destroy(conv_eshard_t e);   /* NULL-safe */

/* Peer-memory exchange (no collective library on the data path): the same steps, but each rank
 * writes its packed U (resp. X) for peer k straight into peer k's receive buffer -- copy-engine
 * transfers over NVLink / NVSwitch between devices, or within one device between processes --
 * at this rank's segment (segments in rank order, the layout forward_b / forward_c read).
 * u_recv_peer[k] / x_recv_peer[k]: the base of rank k's u_recv / x_recv buffer mapped into this
 * process (k == rank: its own buffer), e.g. from conv_ipc_alloc / conv_ipc_open.  The caller
 * orders the ranks: every rank's forward_a_peer (forward_b_peer) must have completed before any
 * rank runs forward_b (forward_c), e.g. stream synchronize + a barrier.  With a tcgen05
 * contraction (not the Gauss epilogue combine) and world <= 8, forward_b_peer's contraction
 * epilogue itself TMA-stores every 32-column X box into its owner's buffer (per-peer tensor
 * maps): the GEMM and the X exchange are one kernel.  The per-image maxima (F16X3) are still
 * gathered by the caller.  Errors: as forward_a / forward_b; INVALID_ARG for a NULL array or
 * entry. */
conv_status conv_eshard_forward_a_peer(conv_eshard_t e, const float *in, const float *w, void *const *u_recv_peer,
                                       float *umax_out, void *workspace, size_t workspace_bytes, void *stream);
conv_status conv_eshard_forward_b_peer(conv_eshard_t e, const void *u_recv, const float *umax_all,
                                       void *const *x_recv_peer, void *workspace, size_t workspace_bytes,
                                       void *stream);

/* Inter-process buffers for the peer exchange: conv_ipc_alloc returns device memory of the
 * current device (cudaMalloc, `bytes` > 0) and its 64-byte IPC handle in handle_out; another
 * process maps it with conv_ipc_open (device pointer valid in that process; peer access enabled
 * lazily) and unmaps it with conv_ipc_close; the owner frees it with conv_ipc_free.  Errors:
 * INVALID_ARG (NULL / zero size), OUT_OF_MEMORY, CUDA. */
conv_status conv_ipc_alloc(size_t bytes, void **ptr, void *handle_out);
conv_status conv_ipc_free(void *ptr);
conv_status conv_ipc_open(const void *handle, void **ptr);
conv_status conv_ipc_close(void *ptr);

#ifdef __cplusplus
}
#endif
#endif /* FASTCONV_H_ */
