// Launchers for the non-GEMM kernels (elementwise, GroupNorm, dual-scope attention core).
// Every launcher returns 0 or a cudaError_t value; none allocates device memory.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace vinf {

int num_sms();
int grid_for(uint64_t work_items, int block);

// ---- elementwise.cu ----
int launch_fill_seeded(void* out, bool bf16, uint64_t n, uint64_t seed, uint64_t first,
                       float scale, cudaStream_t s);
int launch_stub(const void* in, bool in_bf16, uint64_t n, uint32_t C, const float* a,
                const float* c, void* out, bool out_bf16, __nv_bfloat16* hi, __nv_bfloat16* lo,
                cudaStream_t s);
int launch_split(const void* in, bool in_bf16, uint64_t n, __nv_bfloat16* hi, __nv_bfloat16* lo,
                 cudaStream_t s);
int launch_cast(const void* in, bool in_bf16, void* out, bool out_bf16, uint64_t n,
                cudaStream_t s);
// x -= lambda * eps (f64 arithmetic), euler_update_inplace (pipeline.cpp:93-100)
int launch_euler(void* x, const void* eps, bool bf16, uint64_t n, double lambda, cudaStream_t s);

// ---- groupnorm.cu ----
// Scratch needed by launch_group_sums (doubles).
uint64_t group_sums_scratch_elems(uint32_t C);
// sums[g] (+)= sum over the group's elements of x (center == nullptr) or of
// (x - center[g])^2. `accumulate` adds into sums instead of overwriting.
int launch_group_sums(const void* x, bool bf16, uint64_t rows, uint32_t C, uint32_t groups,
                      const double* center, double* sums, double* scratch, bool accumulate,
                      cudaStream_t s);
// stats[g] = sums[g] / count  (count = elements per group, across all clips)
int launch_group_finalize(const double* sums, double count, uint32_t groups, double* stats,
                          cudaStream_t s);
// One pass: sums = [sum x (groups) | sum x^2 (groups)] over the clip (C % 8 == 0, C <= 2048).
// scratch: >= 2 * groups * min(4 * SMs, 512) doubles.
int launch_group_moment_sums(const void* x, bool bf16, uint64_t rows, uint32_t C,
                             uint32_t groups, double* sums, double* scratch, cudaStream_t s);
// Fold per-(32-row block, column) partials fp32 [blocks][2][C] (sum, sum of squares) into
// per-group sums f64 [2][groups], in a fixed order (deterministic).
// scratch: colpart_scratch_elems(C) doubles.
uint64_t colpart_scratch_elems(uint32_t C);
int launch_colpart_to_groups(const float* part, uint32_t blocks, uint32_t C, uint32_t groups,
                             double* sums, double* scratch, cudaStream_t s);
// sums = [sum x (groups) | sum x^2 (groups)] -> stats = [mean | variance]
int launch_group_moments(const double* sums, double count, uint32_t groups, double* stats,
                         cudaStream_t s);
// y = gamma * (x - mean_g) / sqrt(var_g + eps) + beta; optional hi/lo split output.
// count > 0: means holds the whole video's (sum, sum of squares) and vars is unused;
// the moments are formed in the kernel (group_moments_kernel's arithmetic).
// bf16 mode: GroupNorm folded into the next projection W [N][C] (groupnorm.cu):
// wf = bf16(W diag(s)), bias = W t, st = [s; t] (f32, 2C) for the residual affine.
int launch_group_fold(const double* sums, double count, uint32_t C, uint32_t groups, const float* gamma,
                      const float* beta, float eps, const __nv_bfloat16* w, uint32_t N,
                      __nv_bfloat16* wf, float* bias, float* st, cudaStream_t s);
int launch_group_apply(const void* x, bool in_bf16, uint64_t rows, uint32_t C, uint32_t groups,
                       const double* means, const double* vars, const float* gamma,
                       const float* beta, float eps, void* y, bool out_bf16, __nv_bfloat16* hi,
                       __nv_bfloat16* lo, cudaStream_t s, double count = 0.0);

// ---- attention.cu ----
constexpr int kMaxTokens = 160;  // n_local + 1 + n_global upper bound
constexpr int kQBlock = 32;      // queries per tensor-core attention CTA
constexpr int kKvMax = 64;       // distinct K/V frames per query block (tensor-core path)

struct TokenTable {
    const uint16_t* rows;       // [nq][kMaxTokens] key/value frame row (in QKV frame units)
    const uint8_t* biased;      // [nq][kMaxTokens] 1 if this token's logit gets +bias
    const uint16_t* count;      // [nq]
    const uint8_t* col;         // [nq][kMaxTokens] token -> column of its block's K/V list
    const uint16_t* kv_frames;  // [nqb][kKvMax] K/V frame row of each column
    const uint16_t* kv_count;   // [nqb]
    const uint8_t* wlo;         // [nq] first window column of the query's block list
    const uint8_t* whi;         // [nq] last window column (inclusive)
    const uint8_t* gmult;       // [nqb][kKvMax] global tokens on each column
    int wflag, gflag;           // window / global tokens carry +bias
    int kv_ok;                  // every block's K/V list fits kKvMax
    int max_kv;                 // largest K/V list over the blocks
};

// (hi/lo non-null: only the split bf16 planes are written, the fp32-mode GEMM operand)
// ctx[a, p, :] = softmax-attention of query frame a at position p over its token list.
// qkv: [(frames) * HW, 3C] with Q in cols [0,C), K in [C,2C), V in [2C,3C);
// query frame a lives at QKV frame row q_frame0 + a. ctx: [nq * HW, C].
// attention_tc.cu: bf16 tensor-core core (head dim % 64 == 0, <= kKvMax K/V frames per
// 32-query block); launch_attention_core dispatches to it when supported.
bool attention_tc_supported(uint32_t C, uint32_t heads, const TokenTable& tt);
int launch_attention_core_tc(const void* qkv, uint64_t qkv_rows, uint32_t HW, uint32_t C, uint32_t heads, uint32_t nq,
                             uint32_t q_frame0, TokenTable tt, float scale, float bias, void* ctx,
                             cudaStream_t s);

// qkv_rows: rows of the QKV buffer (bounds of the TMA map the bf16 pipeline kernel reads it by)
// attn_fused.cu: Q/K/V projection + attention core in one kernel for clips whose K/V
// tokens are all own frames (the single-worker layout), bf16 mode.
bool fused_attention_supported(uint32_t C, uint32_t heads, uint32_t F, uint32_t HW);
int launch_qkv_attention_fused(const void* u2, uint32_t af, uint32_t f_own0, uint32_t HW, uint32_t C,
                               uint32_t F, const void* wqkv, TokenTable tt, float scale, float bias,
                               void* ctx, cudaStream_t s);

int launch_attention_core(const void* qkv, uint64_t qkv_rows, bool bf16, uint32_t HW, uint32_t C, uint32_t heads,
                          uint32_t nq, uint32_t q_frame0, TokenTable tt, float scale, float bias,
                          void* ctx, bool ctx_bf16, __nv_bfloat16* hi, __nv_bfloat16* lo,
                          cudaStream_t s);

}  // namespace vinf
