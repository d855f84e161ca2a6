// Operator forms over caller-owned device tensors: the reference's single-process ops
// (ops.cpp) and distributed forms (clip_parallel.cpp:194-341), built from the tcgen05
// GEMM, the GroupNorm kernels and the dual-scope attention core.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>

#include "host.hpp"
#include "ops.hpp"

namespace vinf {

void cuda_check(int err, const char* what) {
    if (err != 0)
        throw Error(VINF_ERR, std::string(what) + ": " +
                                  cudaGetErrorString(static_cast<cudaError_t>(err)));
}

int num_sms() {
    static int n = 0;
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
            n = 148;
    });
    return n;
}

// ---- device helpers ----------------------------------------------------------

void DevTokens::upload(const HostTokens& h, cudaStream_t s) {
    const size_t n = h.blob_bytes();
    std::vector<uint8_t> blob(n);
    h.pack(blob.data());
    if (!buf) cuda_check(cudaMallocAsync(&buf, n, s), "cudaMallocAsync(tokens)");
    cuda_check(cudaMemcpyAsync(buf, blob.data(), n, cudaMemcpyHostToDevice, s), "tokens");
    // pageable source: the host blob must outlive the copy
    cuda_check(cudaStreamSynchronize(s), "tokens sync");
    tt = h.view(static_cast<const uint8_t*>(buf));
}

void DevTokens::release() {
    if (buf) cudaFree(buf);
    buf = nullptr;
}

void DevMat::alloc(uint32_t r, uint32_t k) {
    rows = r;
    K = k;
    const size_t n = size_t(r) * k;
    cuda_check(cudaMalloc(&hi, n * 2), "cudaMalloc(weights)");
    cuda_check(cudaMalloc(&lo, n * 2), "cudaMalloc(weights)");
}

void DevMat::from_f32(const float* w_dev, cudaStream_t s) {
    cuda_check(launch_split(w_dev, false, uint64_t(rows) * K, hi, lo, s), "split weights");
}

void DevMat::release() {
    if (hi) cudaFree(hi);
    if (lo) cudaFree(lo);
    hi = lo = nullptr;
}

// ---- GEMM dispatch ------------------------------------------------------------

int g_gemm_debug_flags = 0;

void gemm(const Operand& A, const std::vector<int64_t>& a_rows, const DevMat& B,
          const std::vector<int64_t>& b_rows, int64_t M, int64_t N, const Epilogue& ep, bool split,
          cudaStream_t s) {
    if (A.cols != B.K) shape_error("gemm: K mismatch");
    if (a_rows.size() != b_rows.size() || a_rows.empty()) shape_error("gemm: segment mismatch");
    if (M <= 0 || N <= 0) return;
    if (split && (!A.lo || !B.lo)) shape_error("gemm: split mode needs lo planes");
    const int bn = gemm_pick_block_n(int(N));
    const uint32_t b_box = uint32_t(bn);
    GemmMaps maps;
    std::memset(&maps, 0, sizeof(maps));
    cuda_check(make_tmap_bf16(&maps.a[0], A.hi, A.rows, A.cols, A.ld, 128), "tmap A");
    cuda_check(make_tmap_bf16(&maps.b[0], B.hi, B.rows, B.K, B.K, b_box), "tmap B");
    if (split) {
        cuda_check(make_tmap_bf16(&maps.a[1], A.lo, A.rows, A.cols, A.ld, 128), "tmap A.lo");
        cuda_check(make_tmap_bf16(&maps.b[1], B.lo, B.rows, B.K, B.K, b_box), "tmap B.lo");
    } else {
        maps.a[1] = maps.a[0];
        maps.b[1] = maps.b[0];
    }
    std::vector<GemmSeg> segs;
    for (size_t i = 0; i < a_rows.size(); ++i) {
        const int32_t ar = int32_t(a_rows[i]), br = int32_t(b_rows[i]);
        segs.push_back({0, ar, 0, br});
        if (split) {
            segs.push_back({0, ar, 1, br});
            segs.push_back({1, ar, 0, br});
        }
    }
    // More segments than one launch takes: later launches accumulate through the residual
    // path (res = out), so the TMA residual map (built from ep.res) must not be used, and the
    // partial sums cannot live in split planes.
    const bool chunked = segs.size() > size_t(kGemmMaxSeg);
    if (chunked && ep.out_lo) shape_error("gemm: split-plane output needs <= 12 segments");
    // later chunks re-read the partial sum as their residual: in bf16 that would round it
    if (chunked && ep.out_bf16) shape_error("gemm: bf16 output needs <= 12 segments (taps <= 12)");
    // bf16 output without residual / statistics (the Q/K/V projections): TMA-store epilogue
    const bool tma_out = !chunked && ep.out_bf16 && !ep.res && !ep.colpart && !split &&
                         reinterpret_cast<uintptr_t>(ep.out) % 16 == 0 && ep.out_ld % 8 == 0 &&
                         getenv("VINF_GEMM_NO_TMA_OUT") == nullptr;
    // bf16 output with a bf16 residual and no statistics (the O projection): residual in and
    // output out through TMA (the RT epilogue)
    static const bool no_tma_res = getenv("VINF_GEMM_NO_TMA_RES") != nullptr;
    const bool tma_res = !chunked && ep.out_bf16 && ep.res && ep.res_bf16 && !ep.colpart && !split &&
                         bn % 32 == 0 && reinterpret_cast<uintptr_t>(ep.out) % 16 == 0 &&
                         ep.out_ld % 8 == 0 && reinterpret_cast<uintptr_t>(ep.res) % 16 == 0 &&
                         ep.res_ld % 8 == 0 && !no_tma_res;
    if (tma_out || tma_res)
        cuda_check(make_tmap_out_bf16(&maps.out, ep.out, uint64_t(M), uint64_t(N), uint64_t(ep.out_ld)),
                   "tmap out");
    if (tma_res)
        cuda_check(make_tmap_out_bf16(&maps.res, const_cast<void*>(ep.res), uint64_t(M), uint64_t(N),
                                      uint64_t(ep.res_ld)),
                   "tmap residual");
    // Chunk into launches of <= kGemmMaxSeg segments; later chunks accumulate via the
    // residual path (res = out).
    for (size_t c0 = 0; c0 < segs.size(); c0 += kGemmMaxSeg) {
        GemmParams p;
        std::memset(&p, 0, sizeof(p));
        p.M = int32_t(M);
        p.N = int32_t(N);
        p.K = int32_t(A.cols);
        p.nseg = int32_t(std::min<size_t>(kGemmMaxSeg, segs.size() - c0));
        for (int k = 0; k < p.nseg; ++k) p.seg[k] = segs[c0 + k];
        const bool first = c0 == 0;
        p.bias = first ? ep.bias : nullptr;
        p.res = first ? ep.res : ep.out;
        p.res_scale = first ? ep.res_scale : nullptr;
        p.res_ld = first ? ep.res_ld : ep.out_ld;
        p.res_bf16 = first ? ep.res_bf16 : ep.out_bf16;
        p.out = ep.out;
        p.out_ld = ep.out_ld;
        p.out_bf16 = ep.out_bf16;
        p.out_lo = ep.out_lo;
        p.flags = g_gemm_debug_flags | (tma_out ? kGemmFlagTmaOut : 0) | (tma_res ? kGemmFlagTmaRes : 0);
        if (c0 + kGemmMaxSeg >= segs.size()) p.colpart = ep.colpart;  // final output only
        cuda_check(gemm_tc_launch(maps, p, bn, s), "gemm_tc_launch");
    }
}

// ---- activation operands ------------------------------------------------------

size_t elem_size(vinf_dtype t) { return t == VINF_F32 ? 4 : 2; }

void check_tensor(const vinf_tensor* t, const char* what) {
    if (!t || !t->data) shape_error(std::string(what) + ": null tensor");
    if (t->f == 0 || t->h == 0 || t->w == 0 || t->c == 0)
        shape_error(std::string(what) + ": zero dimension");
    if (t->dtype != VINF_F32 && t->dtype != VINF_BF16) shape_error("unknown dtype");
    if (t->c % 8 != 0)
        shape_error(std::string(what) + ": channels must be a multiple of 8 (16-byte TMA rows)");
}

uint64_t numel(const vinf_tensor* t) { return uint64_t(t->f) * t->h * t->w * t->c; }

TmpBuf::TmpBuf(size_t bytes, cudaStream_t s) : s_(s) {
    if (bytes) cuda_check(cudaMallocAsync(&p, bytes, s), "cudaMallocAsync");
}
TmpBuf::~TmpBuf() {
    if (p) cudaFreeAsync(p, s_);
}

// Operand view of a [rows, C] activation; fp32 inputs are split into hi/lo planes.
ActOperand::ActOperand(const void* data, vinf_dtype dt, uint64_t rows, uint32_t C, cudaStream_t s)
    : planes(dt == VINF_F32 ? rows * C * 4 : 0, s) {
    op.rows = rows;
    op.cols = C;
    op.ld = C;
    if (dt == VINF_BF16) {
        op.hi = static_cast<const __nv_bfloat16*>(data);
        op.lo = nullptr;
    } else {
        auto* hi = static_cast<__nv_bfloat16*>(planes.p);
        auto* lo = hi + rows * C;
        cuda_check(launch_split(data, false, rows * C, hi, lo, s), "split activations");
        op.hi = hi;
        op.lo = lo;
    }
}

// ---- conv ----------------------------------------------------------------------

void conv_over_extended(const vinf_tensor* ext, uint32_t out_start, uint32_t out_len,
                        const vinf_conv_kernel* k, const vinf_tensor* out, cudaStream_t s) {
    check_tensor(ext, "conv input");
    check_tensor(out, "conv output");
    if (!k) shape_error("null conv kernel");
    if (k->C != ext->c) shape_error("conv kernel sized for wrong channel count");
    if (out_len == 0 || out_start > ext->f || out_len > ext->f - out_start)
        range_error("conv output range outside extended tensor");
    if (out->f != out_len || out->h != ext->h || out->w != ext->w || out->c != ext->c)
        shape_error("conv output shape mismatch");
    const uint32_t C = ext->c, hw = ext->h * ext->w;
    const int64_t halo = (k->taps - 1) / 2;
    ActOperand A(ext->data, ext->dtype, uint64_t(ext->f) * hw, C, s);
    std::vector<int64_t> ar, br;
    for (uint32_t j = 0; j < k->taps; ++j) {
        ar.push_back((int64_t(out_start) + int64_t(j) - halo) * hw);  // OOB rows -> zeros
        br.push_back(int64_t(j) * C);
    }
    Epilogue ep;
    ep.bias = k->bias;
    ep.out = out->data;
    ep.out_ld = C;
    ep.out_bf16 = out->dtype == VINF_BF16;
    gemm(A.op, ar, k->w, br, int64_t(out_len) * hw, C, ep, ext->dtype == VINF_F32, s);
}

// ---- group norm ------------------------------------------------------------------

void group_sums(const vinf_tensor* v, uint32_t groups, const double* center, double* sums,
                cudaStream_t s) {
    check_tensor(v, "group norm input");
    if (groups == 0 || v->c % groups != 0) config_error("groups must divide channels");
    TmpBuf scratch(sizeof(double) * group_sums_scratch_elems(v->c), s);
    cuda_check(launch_group_sums(v->data, v->dtype == VINF_BF16, uint64_t(v->f) * v->h * v->w,
                                 v->c, groups, center, sums, static_cast<double*>(scratch.p),
                                 false, s),
               "group sums");
}

void group_stat(const vinf_tensor* v, uint32_t groups, const double* center, double* out,
                cudaStream_t s) {
    TmpBuf sums(sizeof(double) * groups, s);
    group_sums(v, groups, center, static_cast<double*>(sums.p), s);
    const double count = double(numel(v) / groups);
    cuda_check(launch_group_finalize(static_cast<double*>(sums.p), count, groups, out, s),
               "group finalize");
}

void normalize_with_stats(const vinf_tensor* v, const vinf_group_norm_params* p,
                          const double* means, const double* vars, const vinf_tensor* out,
                          cudaStream_t s) {
    check_tensor(v, "group norm input");
    check_tensor(out, "group norm output");
    if (!p || p->groups == 0 || v->c % p->groups != 0)
        config_error("norm groups must divide channels");
    if (!p->gamma || !p->beta) shape_error("group norm params sized for wrong channel count");
    if (!(p->epsilon > 0.0f)) config_error("group norm epsilon must be > 0");
    if (out->f != v->f || out->h != v->h || out->w != v->w || out->c != v->c)
        shape_error("group norm output shape mismatch");
    cuda_check(launch_group_apply(v->data, v->dtype == VINF_BF16, uint64_t(v->f) * v->h * v->w,
                                  v->c, p->groups, means, vars, p->gamma, p->beta, p->epsilon,
                                  out->data, out->dtype == VINF_BF16, nullptr, nullptr, s),
               "group apply");
}

void group_norm(const vinf_tensor* v, const vinf_group_norm_params* p, const vinf_tensor* out,
                cudaStream_t s) {
    if (!p || p->groups == 0 || v->c % p->groups != 0)
        config_error("norm groups must divide channels");
    TmpBuf stats(sizeof(double) * 2 * p->groups, s);
    double* m = static_cast<double*>(stats.p);
    group_stat(v, p->groups, nullptr, m, s);
    group_stat(v, p->groups, m, m + p->groups, s);
    normalize_with_stats(v, p, m, m + p->groups, out, s);
}

// ---- attention ---------------------------------------------------------------------

// Projects `rows` frames of `src` ([rows, hw, C], contiguous) to Q/K/V, runs the core
// for nq queries at frames q0.., projects through Wo into `out`.
void attention_generic(const void* src, vinf_dtype dt, uint32_t frames, uint32_t hw, uint32_t C,
                       uint32_t q0, uint32_t nq, const HostTokens& tok,
                       const vinf_attention_params* p, float bias, const vinf_tensor* out,
                       cudaStream_t s) {
    const bool f32 = dt == VINF_F32;
    const uint64_t rows = uint64_t(frames) * hw;
    ActOperand A(src, dt, rows, C, s);
    // bf16 Q/K/V, or (fp32) the hi and lo bf16 planes of the split arithmetic
    TmpBuf qkv(rows * 3 * C * (f32 ? 4 : 2), s);
    auto* qh = static_cast<__nv_bfloat16*>(qkv.p);
    Epilogue e1;
    e1.out = qh;
    e1.out_lo = f32 ? qh + rows * 3 * C : nullptr;
    e1.out_ld = 3 * C;
    e1.out_bf16 = !f32;
    gemm(A.op, {0}, p->wqkv, {0}, int64_t(rows), 3 * C, e1, f32, s);
    HostTokens tk = tok;
    tk.finalize((C / p->heads) % 64 == 0);
    if (!tk.kv_ok) config_error("a query block touches more than 192 distinct frames");
    if ((C / p->heads) % 8 != 0) config_error("attention head dim (C / heads) must be a multiple of 8");
    DevTokens dt_tok;
    dt_tok.upload(tk, s);
    const uint64_t qrows = uint64_t(nq) * hw;
    TmpBuf ctx(qrows * C * 4, s);  // bf16 ctx or hi+lo planes
    auto* hi = static_cast<__nv_bfloat16*>(ctx.p);
    auto* lo = hi + qrows * C;
    cuda_check(launch_attention_core(qh, f32 ? e1.out_lo : nullptr, frames, hw, C, p->heads, nq, q0, dt_tok.tt,
                                     p->scale, bias, hi, f32 ? lo : nullptr, s),
               "attention core");
    Operand O;
    O.hi = hi;
    O.lo = f32 ? lo : nullptr;
    O.rows = qrows;
    O.cols = C;
    O.ld = C;
    Epilogue e2;
    e2.out = out->data;
    e2.out_ld = C;
    e2.out_bf16 = out->dtype == VINF_BF16;
    gemm(O, {0}, p->wo, {0}, int64_t(qrows), C, e2, f32, s);
    cuda_check(cudaStreamSynchronize(s), "attention sync");  // tokens buffer lifetime
    dt_tok.release();
}

void check_attention(const vinf_tensor* v, const vinf_attention_params* p,
                     const vinf_tensor* out) {
    check_tensor(v, "attention input");
    check_tensor(out, "attention output");
    if (!p) shape_error("null attention params");
    if (p->C != v->c) shape_error("attention dim does not match channels");
    if (out->f != v->f || out->h != v->h || out->w != v->w || out->c != v->c)
        shape_error("attention output shape mismatch");
}

void dual_scope(const vinf_tensor* v, double t, const vinf_attention_params* p,
                const vinf_dual_scope_config* cfg, const vinf_tensor* out, cudaStream_t s) {
    check_attention(v, p, out);
    if (!cfg) shape_error("null dual-scope config");
    const uint32_t F = v->f;
    const auto gset = build_global_index_set(F, cfg->n_global);
    const bool bias_global = t > cfg->t_star;  // ops.cpp:298, strict
    HostTokens tok;
    tok.resize(F);
    for (uint32_t a = 0; a < F; ++a) {
        for (uint32_t g : build_local_window(a, F, cfg->n_local)) tok.push(a, g, !bias_global);
        for (uint32_t g : gset) tok.push(a, g, bias_global, true);
    }
    attention_generic(v->data, v->dtype, F, v->h * v->w, v->c, 0, F, tok, p, cfg->bias, out, s);
}

void attention_full(const vinf_tensor* v, const vinf_attention_params* p, const vinf_tensor* out,
                    cudaStream_t s) {
    check_attention(v, p, out);
    const uint32_t F = v->f;
    if (F > uint32_t(kMaxTokens)) config_error("attention_full supports at most 160 frames");
    HostTokens tok;
    tok.resize(F);
    for (uint32_t a = 0; a < F; ++a)
        for (uint32_t i = 0; i < F; ++i) tok.push(a, i, false);
    attention_generic(v->data, v->dtype, F, v->h * v->w, v->c, 0, F, tok, p, 0.0f, out, s);
}

// ---- distributed forms ------------------------------------------------------------

namespace {
uint32_t frames_of(const vinf_tensor* t) { return (t && t->data) ? t->f : 0; }

// [pre | v | post (| glob)] into one contiguous temporary.
void concat(const std::vector<const vinf_tensor*>& parts, void* dst, size_t fbytes,
            cudaStream_t s) {
    size_t off = 0;
    for (const vinf_tensor* t : parts) {
        const uint32_t f = frames_of(t);
        if (!f) continue;
        cuda_check(cudaMemcpyAsync(static_cast<uint8_t*>(dst) + off, t->data, f * fbytes,
                                   cudaMemcpyDeviceToDevice, s),
                   "concat frames");
        off += f * fbytes;
    }
}
void check_ctx_like(const vinf_tensor* c, const vinf_tensor* v) {
    if (!frames_of(c)) return;
    if (c->h != v->h || c->w != v->w || c->c != v->c || c->dtype != v->dtype)
        shape_error("context frame shape mismatch");
}
}  // namespace

void conv_parallel(uint32_t frames, uint32_t workers, uint32_t worker, const vinf_tensor* v,
                   const vinf_tensor* pre_t, const vinf_tensor* post_t, const vinf_conv_kernel* k,
                   const vinf_tensor* out, cudaStream_t s) {
    check_tensor(v, "conv input");
    const uint32_t f_clip = make_plan(frames, workers);
    if (worker >= workers) range_error("worker index out of range");
    if (v->f != f_clip) protocol_error("clip has wrong frame count for the plan");
    if (!k) shape_error("null conv kernel");
    const uint32_t h = (k->taps - 1) / 2;
    const bool first = worker == 0, last = worker + 1 == workers;
    const uint32_t pre = frames_of(pre_t), post = frames_of(post_t);
    // clip_parallel.cpp:200-206
    if ((first && pre != 0) || (!first && pre != h) || (last && post != 0) || (!last && post != h))
        protocol_error("halo/kernel mismatch on worker " + std::to_string(worker) +
                       ": kernel wants " + std::to_string(h) + " frames per side, got pre=" +
                       std::to_string(pre) + " post=" + std::to_string(post));
    check_ctx_like(pre_t, v);
    check_ctx_like(post_t, v);
    const size_t fb = size_t(v->h) * v->w * v->c * elem_size(v->dtype);
    TmpBuf ext(size_t(pre + f_clip + post) * fb, s);
    concat({pre_t, v, post_t}, ext.p, fb, s);
    vinf_tensor e = *v;
    e.data = ext.p;
    e.f = pre + f_clip + post;
    conv_over_extended(&e, pre, f_clip, k, out, s);
}

void attention_parallel(uint32_t frames, uint32_t workers, uint32_t worker, const vinf_tensor* v,
                        const vinf_tensor* pre_t, const vinf_tensor* post_t,
                        const vinf_tensor* glob_t, double t, const vinf_attention_params* p,
                        const vinf_dual_scope_config* cfg, const vinf_tensor* out,
                        cudaStream_t s) {
    check_attention(v, p, out);
    if (!cfg) shape_error("null dual-scope config");
    const uint32_t f_clip = make_plan(frames, workers);
    if (worker >= workers) range_error("worker index out of range");
    if (v->f != f_clip) protocol_error("clip has wrong frame count for the plan");
    const uint32_t half = cfg->n_local / 2;
    const bool first = worker == 0, last = worker + 1 == workers;
    const uint32_t pre = frames_of(pre_t), post = frames_of(post_t), ng = frames_of(glob_t);
    // clip_parallel.cpp:268-276
    if ((first && pre != 0) || (!first && pre != half) || (last && post != 0) ||
        (!last && post != half) || ng != cfg->n_global)
        protocol_error("context size mismatch on worker " + std::to_string(worker) +
                       ": window needs " + std::to_string(half) + " per side and " +
                       std::to_string(cfg->n_global) + " global frames, got pre=" +
                       std::to_string(pre) + " post=" + std::to_string(post) +
                       " global=" + std::to_string(ng));
    check_ctx_like(pre_t, v);
    check_ctx_like(post_t, v);
    check_ctx_like(glob_t, v);
    const uint32_t ext_f = pre + f_clip + post;
    const uint32_t start = worker * f_clip, ext_start = start - pre;
    const bool bias_global = t > cfg->t_star;
    HostTokens tok;
    tok.resize(f_clip);
    for (uint32_t a = 0; a < f_clip; ++a) {
        for (uint32_t g : build_local_window(start + a, frames, cfg->n_local)) {
            if (g < ext_start || g - ext_start >= ext_f)
                protocol_error("window frame " + std::to_string(g) +
                               " outside synchronized context of worker " +
                               std::to_string(worker));
            tok.push(a, g - ext_start, !bias_global);
        }
        for (uint32_t j = 0; j < cfg->n_global; ++j) tok.push(a, ext_f + j, bias_global, true);
    }
    const size_t fb = size_t(v->h) * v->w * v->c * elem_size(v->dtype);
    TmpBuf ext(size_t(ext_f + ng) * fb, s);
    concat({pre_t, v, post_t, glob_t}, ext.p, fb, s);
    attention_generic(ext.p, v->dtype, ext_f + ng, v->h * v->w, v->c, pre, f_clip, tok, p,
                      cfg->bias, out, s);
}

}  // namespace vinf
