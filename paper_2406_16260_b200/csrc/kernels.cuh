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
// Fold the conv epilogue's column partials fp32 [blocks][2][C] (sum and sum of squares of
// v = u - shift[c], the stored value minus the conv bias) into per-group sums of u, f64
// [2][groups], in a fixed order (deterministic). rows = the rows the partials cover;
// shift may be null (no shift). scratch: colpart_scratch_elems(C) doubles.
uint64_t colpart_scratch_elems(uint32_t C);
int launch_colpart_to_groups(const float* part, uint32_t blocks, uint32_t C, uint32_t groups,
                             const float* shift, double rows, double* sums, double* scratch,
                             cudaStream_t s);
// sums = [sum x (groups) | sum x^2 (groups)] -> stats = [mean | variance]
int launch_group_moments(const double* sums, double count, uint32_t groups, double* stats,
                         cudaStream_t s);
// y = gamma * (x - mean_g) / sqrt(var_g + eps) + beta; optional hi/lo split output.
// count > 0: means holds the whole video's (sum, sum of squares) and vars is unused;
// the moments are formed in the kernel (group_moments_kernel's arithmetic).
// bf16 mode: GroupNorm folded into the next projection W [N][C] (groupnorm.cu):
// wf = bf16(W diag(s)), bias = W t, st = [s; t] (f32, 2C) for the residual affine.
// shift (nullable): the normalised tensor stores u - shift[c]; t absorbs s * shift.
int launch_group_fold(const double* sums, double count, uint32_t C, uint32_t groups, const float* gamma,
                      const float* beta, float eps, const __nv_bfloat16* w, uint32_t N,
                      __nv_bfloat16* wf, float* bias, float* st, const float* shift, cudaStream_t s);
int launch_group_apply(const void* x, bool in_bf16, uint64_t rows, uint32_t C, uint32_t groups,
                       const double* means, const double* vars, const float* gamma,
                       const float* beta, float eps, void* y, bool out_bf16, __nv_bfloat16* hi,
                       __nv_bfloat16* lo, cudaStream_t s, double count = 0.0);

// ---- attention_core.cu ----
constexpr int kMaxTokens = 160;  // n_local + 1 + n_global upper bound
constexpr int kQBlock = 32;      // queries per attention CTA
// distinct K/V frames per 32-query block: the window band (32 + n_local) plus the sampled
// globals never exceeds kQBlock + kMaxTokens - 1 = 191
constexpr int kKvMax = 192;

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
    // TMA load program of each block's K/V list: the sorted distinct frames split into
    // contiguous runs, each run into boxes of <= 32 frame rows (kind = rows - 1), box i
    // packed as frame | smem row << 16 | kind << 24 in kv_box[qb][i] (kv_nbox words); runs of
    // single frames may come as row gathers (kBoxGather4, 3 words). kv_load_rows = the rows
    // those boxes write (= kv_count: the transaction bytes of a K or V stage / 128 B).
    const uint32_t* kv_box;     // [nqb][kKvMax]
    const uint16_t* kv_nbox;    // [nqb]
    const uint16_t* kv_load_rows;  // [nqb]
};
constexpr int kBoxKinds = 32;       // box heights kind + 1 (one TMA op per run of <= 32 frames)
constexpr int kBoxGather4 = 0xFE;   // entry kind: four single frames by one row gather (3 words:
                                    // f0 | row << 16 | kind << 24, f1 | f2 << 16, f3)

// Whether the core runs this configuration: head dim d = C / heads with d % 8 == 0 and
// every query block's distinct K/V frames <= kKvMax. There is no other attention kernel:
// the engine and the operator forms reject what this does not cover.
bool attention_core_supported(uint32_t C, uint32_t heads, const TokenTable& tt);
// ctx[a, p, :] = softmax-attention of query frame a at position p over its token list
// (attend_tokens, ops.cpp:209-241). qkv: [(frames) * HW, 3C] bf16 with Q in cols [0, C),
// K in [C, 2C), V in [2C, 3C); query frame a lives at QKV frame row q_frame0 + a;
// ctx: [nq * HW, C] bf16.
// Split (fp32) mode: qkv_lo / ctx_lo non-null are the lo planes (same layout) of the
// bf16x3 operands; every product runs as hi*hi + hi*lo + lo*hi.
// Fused output (one head, engine.cpp stage_attention): the O projection is absorbed into V
// (the projection emits V' = X (W_o W_v)^T), so ctx' = P V' is already ctx W_o^T and the core
// writes the block output y = ctx' + residual in place of ctx. residual = res * s + t per
// channel (bf16 res, GroupNorm folded: s, t non-null), res (bf16) or res (fp32); y is bf16 or
// fp32 (split mode: from ctx' hi + lo). res and y use ctx's [nq * HW, C] offsets.
struct FuseO {
    const void* res = nullptr;
    const float* s = nullptr;
    const float* t = nullptr;
    void* y = nullptr;  // null: no fusion, ctx is written
    int res_bf16 = 1;
    int y_bf16 = 1;
};
#ifdef __CUDACC__
// v += residual for 8 consecutive channels from `col`, given the raw bf16 residual piece u
__device__ __forceinline__ void fuse_o_add_bf16(const FuseO& f, const uint4& u, uint32_t col, float (&v)[8]) {
    const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&u);
    float r[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float2 x = __bfloat1622float2(u2[k]);
        r[2 * k] = x.x;
        r[2 * k + 1] = x.y;
    }
    if (f.s) {
        const float4 s0 = __ldg(reinterpret_cast<const float4*>(f.s + col));
        const float4 s1 = __ldg(reinterpret_cast<const float4*>(f.s + col) + 1);
        const float4 t0 = __ldg(reinterpret_cast<const float4*>(f.t + col));
        const float4 t1 = __ldg(reinterpret_cast<const float4*>(f.t + col) + 1);
        const float sc[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
        const float tc[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = r[k] * sc[k] + tc[k];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] += r[k];
}
__device__ __forceinline__ void fuse_o_write(const FuseO& f, uint64_t o, const float (&v)[8]) {
    if (f.y_bf16) {
        uint4 w;
        uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const __nv_bfloat162 b2 = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
            wp[k] = *reinterpret_cast<const uint32_t*>(&b2);
        }
        *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(f.y) + o) = w;
    } else {
        float* yf = static_cast<float*>(f.y) + o;
        reinterpret_cast<float4*>(yf)[0] = make_float4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<float4*>(yf)[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
}
// y for 8 consecutive channels from `col` at element offset o, v = ctx' (fp32)
__device__ __forceinline__ void fuse_o_store(const FuseO& f, uint64_t o, uint32_t col, float (&v)[8]) {
    if (f.res_bf16) {
        fuse_o_add_bf16(f, __ldg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(f.res) + o)), col, v);
    } else {
        const float* rf = static_cast<const float*>(f.res) + o;
        const float4 r0 = __ldg(reinterpret_cast<const float4*>(rf));
        const float4 r1 = __ldg(reinterpret_cast<const float4*>(rf) + 1);
        v[0] += r0.x; v[1] += r0.y; v[2] += r0.z; v[3] += r0.w;
        v[4] += r1.x; v[5] += r1.y; v[6] += r1.z; v[7] += r1.w;
    }
    fuse_o_write(f, o, v);
}
// v[8] from one staged 16-byte piece of bf16 (and its lo plane in split mode)
__device__ __forceinline__ void unpack8(const uint4& h, float (&v)[8]) {
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&h);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float2 x = __bfloat1622float2(b[k]);
        v[2 * k] = x.x;
        v[2 * k + 1] = x.y;
    }
}
__device__ __forceinline__ void unpack8_add(const uint4& l, float (&v)[8]) {
    float w[8];
    unpack8(l, w);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] += w[k];
}
#endif
// The same core as a cp.async ring over one position per CTA (attention_cpasync.cu).
int launch_attention_core_cpasync(const void* qkv, const void* qkv_lo, uint32_t HW, uint32_t C, uint32_t heads,
                                  uint32_t nq, uint32_t q_frame0, const TokenTable& tt, float scale, float bias,
                                  void* ctx, void* ctx_lo, cudaStream_t s, const FuseO* fo = nullptr);
// Which implementation launch_attention_core uses: 0 = by configuration, 1 = the TMA ring,
// 2 = the cp.async ring (VINF_ATTN_IMPL=tma|cpasync, vinf_debug_attention_impl).
extern int g_attn_impl;
// qkv_frames: frames of the qkv buffer (the TMA tensor maps' outer extent). fo: fused output
// (null or fo->y null: ctx is written).
int launch_attention_core(const void* qkv, const void* qkv_lo, uint32_t qkv_frames, uint32_t HW, uint32_t C,
                          uint32_t heads, uint32_t nq, uint32_t q_frame0, const TokenTable& tt, float scale,
                          float bias, void* ctx, void* ctx_lo, cudaStream_t s, const FuseO* fo = nullptr);
// out[c][r] = in[r][c] (fp32, rows x cols)
int launch_transpose_f32(const float* in, float* out, uint32_t rows, uint32_t cols, cudaStream_t s);

}  // namespace vinf
