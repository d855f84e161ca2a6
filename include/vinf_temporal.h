/* vinf_temporal.h — C ABI of the B200 (sm_100a) clip-parallel dual-scope temporal block.
 *
 * Drop-in boundary for the reference's temporal-module API. The reference exposes
 * this path only as a C++ API in namespace vinf (/root/reference/proj/src/core/
 * ops.hpp:49-124, clip_parallel.hpp:14-84); its only C ABI (include/vinf.h:27-75) is
 * run-level. Every entry point below names the reference function it replaces.
 *
 * Conventions (mirroring include/vinf.h:1-28 of the reference):
 *   - every function returns a status code; on failure vinf_last_error() holds a
 *     thread-local message valid until the next failing call on the same thread;
 *   - tensors are caller-owned DEVICE buffers in the reference layout [F,H,W,C],
 *     row-major, channels innermost (tensor.hpp:13-24); conv weights [tap][out][in],
 *     projections [out][in] (ops.hpp:11-12); fp32 weights are uploaded once into
 *     parameter handles;
 *   - work is enqueued on the given CUDA stream (cudaStream_t passed as void*);
 *     functions never synchronise the stream unless stated;
 *   - validation happens before any work, as ops.cpp:10-38 does.
 */
#ifndef VINF_TEMPORAL_H
#define VINF_TEMPORAL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: identical values to the reference's vinf.h:18-25. */
enum {
    VINF_OK = 0,
    VINF_ERR = 1,           /* unclassified failure (CUDA errors land here) */
    VINF_ERR_CONFIG = 2,    /* ConfigError: bad taps/groups/halo/plan */
    VINF_ERR_TRANSPORT = 3, /* TransportError / ProtocolError: context size mismatch */
    VINF_ERR_IO = 4,
    VINF_ERR_INVALID = 5,   /* ShapeError / RangeError: bad argument, shape or range */
};

/* Activation storage / arithmetic mode.
 * VINF_F32:  fp32 activations; GEMMs run on tcgen05 as split-bf16 ("bf16x3":
 *            hi*hi + hi*lo + lo*hi, fp32 accumulate); parity bar 1e-4 normwise.
 * VINF_BF16: bf16 activations, bf16 tcgen05 GEMMs, fp32 accumulate/statistics;
 *            parity bar 2e-2 normwise. */
typedef enum { VINF_F32 = 0, VINF_BF16 = 1 } vinf_dtype;

typedef struct {
    void* data;          /* device pointer */
    uint32_t f, h, w, c; /* frames, height, width, channels */
    vinf_dtype dtype;
} vinf_tensor;

const char* vinf_version(void);
const char* vinf_last_error(void);
/* 1 when a CUDA device of compute capability 10.0 is usable, else 0. */
int vinf_device_ok(void);

/* ---- token sets and clip plan (integer-exact host functions) ----------------
 * ops.cpp:177-198, clip_parallel.cpp:54-91, 343-387. `*count` receives the number
 * of entries; `cap` is the capacity of `out`. */
int vinf_build_local_window(uint32_t a, uint32_t frames, uint32_t n_local, uint32_t* out,
                            uint32_t cap, uint32_t* count);
int vinf_build_global_index_set(uint32_t frames, uint32_t n_global, uint32_t* out, uint32_t cap,
                                uint32_t* count);
int vinf_make_plan(uint32_t frames, uint32_t workers, uint32_t* f_clip);
int vinf_global_members_in_range(uint32_t frames, uint32_t n_global, uint32_t start,
                                 uint32_t len, uint32_t* out, uint32_t cap, uint32_t* count);
/* out[3] = {bytes_sent, bytes_contributed, messages} (TrafficPrediction). */
int vinf_predict_sync_traffic(uint32_t frames, uint32_t workers, uint32_t halo,
                              uint32_t global_frames, uint32_t worker, uint64_t frame_bytes,
                              uint64_t* out3);
int vinf_predict_groupnorm_traffic(uint32_t frames, uint32_t workers, uint32_t groups,
                                   uint32_t worker, uint64_t* out3);

/* ---- synthetic inputs and random-init weights (bit-exact on device) ----------
 * tensor_from_seed_at (tensor.cpp:98-106) and draw() (pipeline.cpp:26-31):
 * dst[i] = unit(seed, first_elem + i) * scale, rounded to dtype. */
int vinf_fill_seeded(void* dst, vinf_dtype dtype, uint64_t n, uint64_t seed, uint64_t first_elem,
                     float scale, void* stream);
uint64_t vinf_mix_seed(uint64_t seed, uint64_t salt); /* rng.hpp:34-37 */

/* ---- parameter handles ------------------------------------------------------- */
/* ConvKernel (ops.hpp:14-21). weights: taps*C*C fp32, bias: C fp32, both DEVICE. */
typedef struct vinf_conv_kernel vinf_conv_kernel;
int vinf_conv_kernel_create(uint32_t taps, uint32_t channels, const float* weights,
                            const float* bias, vinf_conv_kernel** out);
void vinf_conv_kernel_destroy(vinf_conv_kernel* k);

/* AttentionParams (ops.hpp:32-36) + a heads extension (heads == 1 is the
 * reference: head dim == C). wq/wk/wv/wo: C*C fp32 DEVICE. */
typedef struct vinf_attention_params vinf_attention_params;
int vinf_attention_params_create(uint32_t dim, uint32_t heads, float scale, const float* wq,
                                 const float* wk, const float* wv, const float* wo,
                                 vinf_attention_params** out);
void vinf_attention_params_destroy(vinf_attention_params* p);

/* GroupNormParams (ops.hpp:23-30); gamma/beta are C fp32 DEVICE pointers. */
typedef struct {
    uint32_t groups;
    const float* gamma;
    const float* beta;
    float epsilon;
} vinf_group_norm_params;

/* DualScopeConfig (ops.hpp:38-43). */
typedef struct {
    uint32_t n_local;
    uint32_t n_global;
    float bias;
    double t_star;
} vinf_dual_scope_config;

/* ---- operators (reference single-process forms) ------------------------------ */
/* spatial_affine_tanh (ops.cpp:42-55); a, c: C fp32 device. */
int vinf_spatial_affine_tanh(const vinf_tensor* v, const float* a, const float* c,
                             vinf_tensor* out, void* stream);
/* conv_over_extended (ops.cpp:73-104): out frames [out_start, out_start+out_len) of ext;
 * frames outside [0, ext.f) are zeros. out: [out_len,H,W,C]. */
int vinf_conv_over_extended(const vinf_tensor* ext, uint32_t out_start, uint32_t out_len,
                            const vinf_conv_kernel* k, vinf_tensor* out, void* stream);
/* temporal_conv (ops.cpp:106-108) */
int vinf_temporal_conv(const vinf_tensor* v, const vinf_conv_kernel* k, vinf_tensor* out,
                       void* stream);
/* group_means / group_sqdev (ops.cpp:112-142): f64 DEVICE outputs [groups]. */
int vinf_group_means(const vinf_tensor* v, uint32_t groups, double* means, void* stream);
int vinf_group_sqdev(const vinf_tensor* v, uint32_t groups, const double* means, double* vars,
                     void* stream);
/* Partial sums for the distributed form: sums[g] = sum x (center == NULL) or
 * sum (x - center[g])^2 over this clip. f64 DEVICE. */
int vinf_group_partial_sums(const vinf_tensor* v, uint32_t groups, const double* center,
                            double* sums, void* stream);
/* normalize_with_stats (ops.cpp:144-167); means/vars f64 DEVICE. */
int vinf_normalize_with_stats(const vinf_tensor* v, const vinf_group_norm_params* p,
                              const double* means, const double* vars, vinf_tensor* out,
                              void* stream);
/* group_norm (ops.cpp:169-173) */
int vinf_group_norm(const vinf_tensor* v, const vinf_group_norm_params* p, vinf_tensor* out,
                    void* stream);
/* dual_scope_reference (ops.cpp:291-338); attention_full (ops.cpp:264-289). */
int vinf_dual_scope_attention(const vinf_tensor* v, double t, const vinf_attention_params* p,
                              const vinf_dual_scope_config* cfg, vinf_tensor* out, void* stream);
int vinf_attention_full(const vinf_tensor* v, const vinf_attention_params* p, vinf_tensor* out,
                        void* stream);

/* ---- distributed operator forms (clip_parallel.cpp:194-341) -------------------
 * ctx_pre / ctx_post: the neighbours' boundary frames (NULL or f == 0 at the video
 * edge); ctx_global: the n_global gathered frames in global-index order. Context
 * sizes are checked exactly as the reference does (ProtocolError ->
 * VINF_ERR_TRANSPORT). */
int vinf_conv_parallel(uint32_t frames, uint32_t workers, uint32_t worker, const vinf_tensor* v,
                       const vinf_tensor* ctx_pre, const vinf_tensor* ctx_post,
                       const vinf_conv_kernel* k, vinf_tensor* out, void* stream);
int vinf_attention_parallel(uint32_t frames, uint32_t workers, uint32_t worker,
                            const vinf_tensor* v, const vinf_tensor* ctx_pre,
                            const vinf_tensor* ctx_post, const vinf_tensor* ctx_global, double t,
                            const vinf_attention_params* p, const vinf_dual_scope_config* cfg,
                            vinf_tensor* out, void* stream);

/* ---- clip engine: the fused, preallocated block stack of one worker -----------
 * eps_theta_worker (pipeline.cpp:145-172) for `blocks` blocks on one clip, with all
 * buffers (halo slots, global slots, Q/K/V, statistics) carved from ONE caller-owned
 * device workspace. Cross-worker context moves (the paper's 3-step sync) are exposed
 * as exchange lists of (peer, direction, workspace offset, bytes) so the caller's
 * transport (NCCL via torch.distributed, or in-process copies) executes them between
 * stages; with one worker every list is empty and vinf_engine_forward runs the whole
 * stack in one call. */
typedef struct {
    uint32_t frames, workers, worker;
    uint32_t height, width, channels;
    uint32_t taps, groups, heads;
    uint32_t n_local, n_global;
    float bias;
    double t_star;
    float epsilon;
    float scale;        /* 0 -> 1/sqrtf(C/heads) */
    uint32_t blocks;
    vinf_dtype dtype;
    /* Extension (not in the reference, which needs workers | frames, clip_parallel.cpp:56-59):
     * 1 = uneven clips, worker w owning frames [floor(w*F/N), floor((w+1)*F/N)), e.g. the
     * paper's 2,300 frames over 8 GPUs. 0 = the reference's even split. */
    uint32_t uneven;
} vinf_engine_desc;

typedef struct vinf_layout vinf_layout;
/* Pure host: buffer layout + exchange plan. No CUDA calls (usable on CPU hosts). */
int vinf_layout_create(const vinf_engine_desc* d, vinf_layout** out);
void vinf_layout_destroy(vinf_layout* l);
int vinf_layout_workspace_bytes(const vinf_layout* l, uint64_t* bytes);
/* This worker's clip: first global frame and frame count. */
int vinf_layout_clip(const vinf_layout* l, uint32_t* start, uint32_t* frames);

/* Named regions of the workspace (for the caller's views / tests). */
enum {
    VINF_BUF_X = 0,      /* block input  [f_clip,H,W,C] dtype */
    VINF_BUF_Y = 1,      /* block output [f_clip,H,W,C] dtype */
    VINF_BUF_CONV_IN = 2,/* conv operand, frames [hc | f_clip | hc] (bf16 plane / hi plane) */
    VINF_BUF_ATTN_IN = 3,/* attention operand, frames [ha | f_clip | ha | remote globals] */
    VINF_BUF_GN_SUMS = 4,/* f64 [2][groups] */
    VINF_BUF_QKV = 5,    /* [attn frames * H*W, 3C] engine dtype (Q | K | V per row); with one
                            head the V columns hold V' = X (W_o W_v)^T (the O projection absorbed) */
    VINF_BUF_CTX = 6     /* [f_clip * H*W, C] attention context (bf16 / hi plane); not written with
                            one head, where the core writes the block output (VINF_NO_FUSE_O=1: it is) */
};
int vinf_layout_region(const vinf_layout* l, int which, uint64_t* offset, uint64_t* bytes,
                       uint64_t* frame_bytes);

/* Exchange stages. */
enum { VINF_XCHG_CONV = 0, VINF_XCHG_ATTN = 1 };
typedef struct {
    uint32_t peer;
    uint32_t send;      /* 1 = send to peer, 0 = receive from peer */
    uint32_t tag;       /* matching key: identical on both ends of one message */
    uint32_t reserved;
    uint64_t offset;    /* workspace byte offset */
    uint64_t bytes;
} vinf_xfer;
/* Transfers of one exchange stage in a deadlock-free order (every send has exactly one
 * matching receive with the same tag on the peer). out = NULL with cap = 0 only sets
 * *count (size query). */
int vinf_layout_exchange(const vinf_layout* l, int stage, vinf_xfer* out, uint32_t cap,
                         uint32_t* count);
/* Logical bytes the reference's sync would move for this worker per block
 * (predict_sync_traffic for conv + attention, predict_groupnorm_traffic). */
int vinf_layout_reference_traffic(const vinf_layout* l, uint64_t* conv3, uint64_t* gn3,
                                  uint64_t* attn3);

typedef struct vinf_engine vinf_engine;
/* workspace: DEVICE buffer of vinf_layout_workspace_bytes bytes (zeroed by create). */
int vinf_engine_create(const vinf_layout* l, void* workspace, void* stream, vinf_engine** out);
void vinf_engine_destroy(vinf_engine* e);
/* Block b's weights from fp32 DEVICE buffers in the reference layout. */
int vinf_engine_set_block(vinf_engine* e, uint32_t block, const float* stub_a,
                          const float* stub_c, const float* conv_w, const float* conv_b,
                          const float* gamma, const float* beta, const float* wq,
                          const float* wk, const float* wv, const float* wo, void* stream);
/* build_model (pipeline.cpp:35-67) on device for every block. */
int vinf_engine_init_weights(vinf_engine* e, uint64_t weight_seed, void* stream);

/* Stages of one block (between them the caller runs the exchanges):
 *   STUB      : x -> u0 (conv operand centre)                 then VINF_XCHG_CONV
 *   CONV      : u1 = u0 + conv(u0), with the clip's GroupNorm (sum, sum of squares)
 *               per group fused into the GEMM epilogue            then all-reduce GN_SUMS
 *   GN_APPLY  : mean/var from the all-reduced sums; u2 = GN(u1)  then VINF_XCHG_ATTN
 *   ATTENTION : y = u2 + dual_scope(u2, t)  (y becomes the next block's x)
 * (The reference combines GN statistics in two rounds, clip_parallel.cpp:242-253; the
 * engine needs one all-reduce of 2*groups doubles; op-level vinf_group_norm keeps the
 * reference's two-pass arithmetic.) */
enum {
    VINF_STAGE_STUB = 0,
    VINF_STAGE_CONV = 1,
    VINF_STAGE_GN_APPLY = 2,
    VINF_STAGE_ATTENTION = 3,
    /* Optional split of ATTENTION: the own frames' Q/K/V projection, which needs no
     * exchanged frame, so it can run while the attention exchange is in flight; the
     * following ATTENTION stage then skips it. */
    VINF_STAGE_QKV = 4
};
int vinf_engine_stage(vinf_engine* e, uint32_t block, int stage, double t, void* stream);
/* All blocks, all stages (single worker: no exchanges needed). */
int vinf_engine_forward(vinf_engine* e, double t, void* stream);
/* Where the clip x (block-stack input, never overwritten by the blocks) and the stack's
 * output y (= eps) live (device pointers). */
int vinf_engine_io(const vinf_engine* e, void** x, void** y);
/* euler_update_inplace (pipeline.cpp:93-100): x -= lambda * y. */
int vinf_engine_euler(vinf_engine* e, double lambda, void* stream);
/* Sync ablation (the reference's `ablate` run key, pipeline.cpp:150-170; values are its
 * LayerKind numbers, metrics.hpp:11). The driver must skip that kind's exchange (or the
 * all-reduce, for groupnorm); the engine then uses zero context frames (conv: halo
 * slots; attention: halo + remote global slots) or clip-local GroupNorm statistics. */
enum {
    VINF_ABLATE_NONE = 0,
    VINF_ABLATE_CONV = 1,
    VINF_ABLATE_GROUPNORM = 2,
    VINF_ABLATE_ATTENTION = 3
};
int vinf_engine_set_ablation(vinf_engine* e, int kind);
/* worker_denoise (pipeline.cpp:174-191) for one worker: for t in timestep_grid(steps)
 * (1000 j / steps, j = steps..1): y = eps_theta(x, t); x -= y / steps. Result in x. */
int vinf_engine_denoise(vinf_engine* e, uint32_t steps, void* stream);
/* Number of kernel launches this engine has enqueued so far. */
uint64_t vinf_engine_launches(const vinf_engine* e);
/* Per-kernel timing: with profiling on, CUDA events are recorded on the launching
 * stream around each kernel group; vinf_engine_kernel_stats synchronises on them and
 * returns, per kernel name (comma-separated in `names`), the summed milliseconds and
 * the launch count since the last read, then resets. */
int vinf_engine_profile(vinf_engine* e, int enable);
int vinf_engine_kernel_stats(vinf_engine* e, char* names, uint32_t name_cap, double* total_ms,
                             uint64_t* counts, uint32_t cap, uint32_t* n_out);

/* ---- clip-parallel executor: the paper's 3-step context sync in C++ ------------
 * Replaces the reference's Transport (transport.hpp:20-43: point-to-point messages
 * matched by (peer, tag) plus the GroupNorm statistics exchange) and its worker loop
 * eps_theta_worker (pipeline.cpp:145-172) + sync_contexts (clip_parallel.cpp:93-192).
 * One communicator per worker:
 *   vinf_comm_create_nccl  : NCCL over NVLink / NVSwitch, one process (or thread) per GPU;
 *                            every rank passes the id rank 0 got from
 *                            vinf_comm_nccl_unique_id (distributed out of band);
 *   vinf_comm_create_local : N in-process workers (threads; device copies between their
 *                            workspaces, the all-reduce summed in worker order), the
 *                            shape of run_inproc_workers (transport_inproc.cpp:148-189);
 *   vinf_comm_create_ops   : caller callbacks (any transport; pointers are whatever the
 *                            exchanged workspace is: device memory, or host memory when
 *                            a plan is run on a CPU host with vinf_layout_run_exchange). */
typedef struct vinf_comm vinf_comm;
typedef struct {
    void* ctx;
    /* optional: bracket the messages of one exchange; all must be complete (in stream
     * order) when group_end returns */
    int (*group_start)(void* ctx);
    int (*send)(void* ctx, uint32_t peer, uint32_t tag, const void* ptr, uint64_t bytes, void* stream);
    int (*recv)(void* ctx, uint32_t peer, uint32_t tag, void* ptr, uint64_t bytes, void* stream);
    int (*group_end)(void* ctx, void* stream);
    /* in-place sum over all ranks, identical result on every rank */
    int (*allreduce_sum_f64)(void* ctx, double* ptr, uint64_t count, void* stream);
} vinf_transport_ops;
int vinf_comm_nccl_unique_id(uint8_t id[128]);
/* Collective over the ranks: binds the communicator to the CURRENT CUDA device. */
int vinf_comm_create_nccl(const uint8_t id[128], uint32_t nranks, uint32_t rank, vinf_comm** out);
/* out: array of nranks communicators sharing one in-process hub (one per worker thread). */
int vinf_comm_create_local(uint32_t nranks, vinf_comm** out);
int vinf_comm_create_ops(const vinf_transport_ops* ops, uint32_t nranks, uint32_t rank, vinf_comm** out);
void vinf_comm_destroy(vinf_comm* c);
/* In-process workers: wakes every worker blocked in an exchange of this hub with a
 * VINF_ERR_TRANSPORT error (call it when one worker fails). No-op for other kinds. */
void vinf_comm_abort(vinf_comm* c);
int vinf_comm_info(const vinf_comm* c, uint32_t* nranks, uint32_t* rank, uint64_t* bytes_sent,
                   uint64_t* messages_sent);
int vinf_comm_allreduce_sum_f64(vinf_comm* c, double* ptr, uint64_t count, void* stream);
/* Runs one exchange stage of a layout's plan over `comm`, `base` = the workspace (pure
 * host logic + the communicator's calls: usable on a CPU host with an ops transport). */
int vinf_layout_run_exchange(const vinf_layout* l, int stage, void* base, vinf_comm* comm, void* stream);
/* The engine's exchanges / GroupNorm all-reduce over a communicator, on `stream`. */
int vinf_engine_exchange(vinf_engine* e, int stage, vinf_comm* comm, void* stream);
int vinf_engine_allreduce_sums(vinf_engine* e, vinf_comm* comm, void* stream);
/* One worker's whole block stack with the 3-step sync, all in C++ (the caller's thread
 * only enqueues): per block
 *   stub of the clip's boundary frames -> conv halo exchange on the engine's comm stream
 *     || stub of the interior frames;
 *   conv (+ GroupNorm partial sums) -> all-reduce of the 2*groups sums;
 *   GroupNorm fold / apply -> attention halo + remote-global exchange on the comm stream
 *     || the own frames' Q/K/V projection;
 *   halo / remote-global K/V projection, attention core, O projection + residual.
 * Exchanges of the kind set with vinf_engine_set_ablation are skipped. With an NCCL
 * communicator the stack of each timestep regime is captured into a CUDA graph once
 * and replayed (use_graph != 0). Every worker must call it with the same t. */
int vinf_engine_forward_dist(vinf_engine* e, double t, vinf_comm* comm, int use_graph, void* stream);
/* worker_denoise (pipeline.cpp:174-191) over the communicator. */
int vinf_engine_denoise_dist(vinf_engine* e, uint32_t steps, vinf_comm* comm, int use_graph, void* stream);

/* ---- diagnostics ---------------------------------------------------------------
 * Times the segmented tcgen05 GEMM alone on synthetic bf16 data: out[M,N] (bf16) =
 * sum over nseg segments of A[M,K] B[N,K]^T (+ bf16 residual); flags = 1 skips the
 * epilogue's global stores (isolates the main loop). Average ms over iters launches. */
int vinf_gemm_bench(uint32_t M, uint32_t N, uint32_t K, uint32_t nseg, int flags, int residual,
                    int iters, float* avg_ms);
/* The attention core alone on a single-worker engine layout's token table (t > t_star),
 * over a synthetic Q/K/V buffer; pos_major must be 0 (frame-major; the position-major and
 * chunked layouts were measured and removed). */
int vinf_attention_bench(uint32_t frames, uint32_t height, uint32_t width, uint32_t channels, uint32_t heads,
                         uint32_t n_local, uint32_t n_global, int f32, int pos_major, int iters, float* avg_ms);
/* The attention core's feed for later launches: 0 = by configuration (TMA ring for bf16
 * blocks of <= 32 distinct K/V frames, cp.async ring otherwise), 1 = TMA ring, 2 = cp.async
 * ring. Returns the previous setting. */
int vinf_debug_attention_impl(int impl);
/* Streaming 16-byte loads over `bytes` of device memory. */
int vinf_read_bw_bench(uint64_t bytes, int iters, float* avg_ms);
/* 1-D bulk copies (TMA) of `chunk` bytes into an mbarrier ring of `stages` slots per CTA,
 * `ctas` CTAs per SM (the attention core's feed without its compute). */
int vinf_bulk_bw_bench(uint64_t bytes, uint32_t chunk, uint32_t stages, uint32_t ctas, int iters, float* avg_ms);

#ifdef __cplusplus
}
#endif

#endif /* VINF_TEMPORAL_H */
