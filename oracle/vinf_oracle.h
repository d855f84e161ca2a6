/* CPU restatement of the reference temporal-block path — TEST INFRASTRUCTURE ONLY.
 *
 * This header and vinf_oracle.c restate, in plain C, the algorithms of the
 * reference C++ library (/root/reference/proj/src/core/{ops,clip_parallel,
 * pipeline,tensor,rng}.*) that the B200 product path replaces. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it; the
 * product (paper_2406_16260_b200/) never links or calls it.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against
 *   (1) the golden vectors frozen in the reference's own tests
 *       (test_tensor.cpp:57-61, test_ops.cpp:302-354, test_clip_parallel.cpp:66-81), and
 *   (2) the reference itself, compiled from its sources by oracle/Makefile into
 *       oracle/_ref/libvinf_ref.so (bitwise on the same host).
 *
 * All layouts follow the reference: activations [F,H,W,C] fp32 row-major with
 * channels innermost (tensor.hpp:13-24), conv weights [tap][out][in], projections
 * [out][in] (ops.hpp:11-12). Accumulation is f64 and stores are f32, exactly as
 * ops.cpp does.
 */
#ifndef VINF_ORACLE_H
#define VINF_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* rng.hpp:14-19 / :23-26 / :34-37 */
uint64_t orc_splitmix_next(uint64_t* state);
float orc_next_unit(uint64_t* state);
uint64_t orc_mix_seed(uint64_t seed, uint64_t salt);
/* tensor.cpp:98-106: element i of the stream entered at first_elem */
void orc_fill_seeded(float* out, size_t n, uint64_t seed, uint64_t first_elem, float scale);

/* pipeline.cpp:35-67 — one block's parameters. Buffers are caller-owned:
 * stub_a/stub_c [C], conv_w [taps*C*C], conv_b [C], gamma/beta [C],
 * wq/wk/wv/wo [C*C]. */
int orc_build_block(uint32_t channels, uint32_t taps, uint64_t weight_seed, uint32_t block,
                    float* stub_a, float* stub_c, float* conv_w, float* conv_b, float* gamma,
                    float* beta, float* wq, float* wk, float* wv, float* wo);

/* ops.cpp:42-55 */
void orc_spatial_affine_tanh(const float* v, size_t n, uint32_t C, const float* a, const float* c,
                             float* out);

/* ops.cpp:73-104: ext is [ext_f,H,W,C]; out is [out_len,H,W,C]. Returns 0 or an
 * error code (1 config, 2 range). */
int orc_conv_over_extended(const float* ext, uint32_t ext_f, uint32_t H, uint32_t W, uint32_t C,
                           uint32_t out_start, uint32_t out_len, uint32_t taps, const float* wts,
                           const float* bias, float* out);

/* ops.cpp:112-173 */
int orc_group_means(const float* v, size_t total, uint32_t C, uint32_t groups, double* means);
int orc_group_sqdev(const float* v, size_t total, uint32_t C, uint32_t groups,
                    const double* means, double* vars);
int orc_normalize_with_stats(const float* v, size_t total, uint32_t C, uint32_t groups,
                             const float* gamma, const float* beta, float eps,
                             const double* means, const double* vars, float* out);
int orc_group_norm(const float* v, size_t total, uint32_t C, uint32_t groups, const float* gamma,
                   const float* beta, float eps, float* out);

/* ops.cpp:177-198. Return the count written (or -1 on error). */
int orc_build_local_window(uint32_t a, uint32_t frames, uint32_t n_local, uint32_t* out);
int orc_build_global_index_set(uint32_t frames, uint32_t n_global, uint32_t* out);

/* ops.cpp:200-207 */
void orc_project_vec(const float* w, const float* x, uint32_t dim, float* y);

/* ops.cpp:264-289 (full attention, optional row sums per (position, query)) */
int orc_attention_full(const float* v, uint32_t F, uint32_t H, uint32_t W, uint32_t C,
                       const float* wq, const float* wk, const float* wv, const float* wo,
                       float scale, float* out, double* row_sums);

/* ops.cpp:291-338. heads > 1 is an EXTENSION not pinned by the reference
 * (the reference is single-head, dim == C, ops.hpp:33): each head h uses
 * channels [h*C/heads, (h+1)*C/heads) of q/k/v, the same token list/bias and
 * `scale`; heads == 1 is exactly the reference. counters (optional, 3 u64):
 * score_entries, queries, max_tokens_per_query (ops.hpp:98-102). */
int orc_dual_scope(const float* v, uint32_t F, uint32_t H, uint32_t W, uint32_t C, double t,
                   const float* wq, const float* wk, const float* wv, const float* wo, float scale,
                   uint32_t heads, uint32_t n_local, uint32_t n_global, float bias, double t_star,
                   float* out, uint64_t* counters);

/* clip_parallel.cpp:256-341 restricted to one worker. v: [f_clip,H,W,C];
 * pre/post: [n_local/2,H,W,C] or NULL at the video edge; glob: [n_global,H,W,C]. */
int orc_attention_parallel(uint32_t frames, uint32_t workers, uint32_t worker, const float* v,
                           const float* pre, const float* post, const float* glob, uint32_t H,
                           uint32_t W, uint32_t C, double t, const float* wq, const float* wk,
                           const float* wv, const float* wo, float scale, uint32_t heads,
                           uint32_t n_local, uint32_t n_global, float bias, double t_star,
                           float* out);

/* clip_parallel.cpp:54-91, 343-387 */
int orc_make_plan(uint32_t frames, uint32_t workers, uint32_t* f_clip);
int orc_global_members_in_range(uint32_t frames, uint32_t n_global, uint32_t start, uint32_t len,
                                uint32_t* out);
/* out[3] = bytes_sent, bytes_contributed, messages */
int orc_predict_sync_traffic(uint32_t frames, uint32_t workers, uint32_t halo,
                             uint32_t global_frames, uint32_t worker, uint64_t frame_bytes,
                             uint64_t* out);
int orc_predict_groupnorm_traffic(uint32_t frames, uint32_t workers, uint32_t groups,
                                  uint32_t worker, uint64_t* out);

/* pipeline.cpp:102-111 for one block: stub -> u + conv(u) -> GN -> u + attn(u, t).
 * x and out: [F,H,W,C]. Params as orc_build_block. */
int orc_block_forward(const float* x, uint32_t F, uint32_t H, uint32_t W, uint32_t C,
                      uint32_t taps, uint32_t groups, double t, const float* stub_a,
                      const float* stub_c, const float* conv_w, const float* conv_b,
                      const float* gamma, const float* beta, float eps, const float* wq,
                      const float* wk, const float* wv, const float* wo, float scale,
                      uint32_t heads, uint32_t n_local, uint32_t n_global, float bias,
                      double t_star, float* out);

#ifdef __cplusplus
}
#endif

#endif
