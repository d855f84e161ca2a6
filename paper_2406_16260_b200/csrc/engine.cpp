// Clip engine: eps_theta_worker (pipeline.cpp:145-172) for one worker's clip, with every
// activation buffer carved from one preallocated workspace (layout.hpp) and every
// kernel enqueued on the caller's stream. The 3-step context sync happens between
// stages through exchange lists (plan.cpp), executed by the caller's transport.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>

#include "comm.hpp"
#include "host.hpp"
#include "layout.hpp"
#include "ops.hpp"

namespace vinf {

enum ParamSlot : uint64_t {  // pipeline.cpp:16-26
    kStub = 0, kConvW = 1, kConvB = 2, kGamma = 3, kBeta = 4, kWq = 5, kWk = 6, kWv = 7, kWo = 8
};

uint64_t mix_seed(uint64_t seed, uint64_t salt) {  // rng.hpp:34-37
    uint64_t z = (seed ^ (salt * 0xD1B54A32D192ED03ull)) + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

}  // namespace vinf

using namespace vinf;

struct EngineBlock {
    float* f32 = nullptr;  // one allocation: stub_a, stub_c, conv_b, gamma, beta (5*C)
    float* stub_a() const { return f32; }
    float* stub_c() const { return f32 + C; }
    float* conv_b() const { return f32 + 2 * C; }
    float* gamma() const { return f32 + 3 * C; }
    float* beta() const { return f32 + 4 * C; }
    uint32_t C = 0;
    DevMat conv;  // [taps*C, C]
    DevMat wqkv;  // [3C, C]; with one head its V rows hold W_o W_v, re-formed every step
    DevMat wo;    // [C, C]
    DevMat wvT;   // [C, C]: W_v transposed, the B operand of W_o W_v
};

struct vinf_engine {
    explicit vinf_engine(const Layout& l) : L(l) {}
    Layout L;
    uint8_t* ws = nullptr;
    std::vector<EngineBlock> blocks;
    TokenTable tt[4];  // [ablated attention sync * 2 + bias_global]
    uint64_t launches = 0;

    // The single-worker block stack is a fixed launch sequence per timestep regime (the
    // only t dependence is the strict t > t_star bias flag, ops.cpp:298), so it is captured
    // once per regime into a CUDA graph and replayed: no per-kernel launch gaps. Captured
    // on a private stream (the caller's may be the legacy stream), launched on the caller's.
    struct Graph {
        cudaGraphExec_t exec = nullptr;
        uint64_t nlaunch = 0, nbytes = 0, nmsgs = 0;
        int calls = 0;
    };
    Graph graphs[2];
    cudaStream_t cap_stream = nullptr;
    // Clip-parallel executor (vinf_engine_forward_dist): the exchanges run on a side
    // stream, ordered against the compute stream by events; the exchange lists are sorted
    // once into the order both ends of a message pair post them.
    struct Dist {
        cudaStream_t cs = nullptr;
        cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
        std::vector<vinf_xfer> xconv, xattn;
        Graph graphs[2];
        const vinf_comm* graph_comm = nullptr;
    } dist;
    void dist_init();
    void dist_block(uint32_t b, double t, vinf_comm* comm, cudaStream_t s);
    bool use_graphs = getenv("VINF_NO_GRAPH") == nullptr;
    void drop_graphs() {
        for (Graph* gs : {graphs, dist.graphs})
            for (int i = 0; i < 2; ++i) {
                if (gs[i].exec) cudaGraphExecDestroy(gs[i].exec);
                gs[i] = Graph{};
            }
        dist.graph_comm = nullptr;
    }

    // Optional per-kernel timing: CUDA events recorded on the launching stream around
    // each kernel (group), aggregated by name on request (vinf_engine_kernel_stats).
    bool profiling = false;
    struct Rec { const char* name; cudaEvent_t a, b; };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    size_t pool_used = 0;
    cudaEvent_t ev() {
        if (pool_used == pool.size()) {
            cudaEvent_t e;
            cuda_check(cudaEventCreate(&e), "cudaEventCreate");
            pool.push_back(e);
        }
        return pool[pool_used++];
    }
    struct Span {
        vinf_engine* e;
        const char* name;
        cudaStream_t s;
        cudaEvent_t a = nullptr;
        Span(vinf_engine* eng, const char* n, cudaStream_t st) : e(eng), name(n), s(st) {
            if (e->profiling) {
                a = e->ev();
                cudaEventRecord(a, s);
            }
        }
        ~Span() {
            if (a) {
                cudaEvent_t b = e->ev();
                cudaEventRecord(b, s);
                e->recs.push_back({name, a, b});
            }
        }
    };

    template <class T = uint8_t>
    T* at(uint64_t off) const { return reinterpret_cast<T*>(ws + off); }
    bool f32() const { return L.f32; }
    uint64_t clip_elems() const { return uint64_t(L.f_clip) * L.E; }
    // Block b writes Y if an even number of blocks follow it, else TMP, so the last block
    // always writes Y and X (the clip being denoised) is never overwritten.
    void* y_of(uint32_t b) const {
        return at((blocks.size() - 1 - b) % 2 == 0 ? L.off_y : L.off_tmp);
    }
    void* x_of(uint32_t b) const { return b == 0 ? at(L.off_x) : y_of(b - 1); }
    double gn_count() const {  // elements per group over the whole video (or the clip)
        const uint64_t f = ablate == VINF_ABLATE_GROUPNORM ? L.f_clip : L.d.frames;
        return double(f * L.hw * L.d.channels / L.d.groups);
    }

    // Sync ablation (pipeline.cpp:150-170 with `ablate`): the driver skips that kind's
    // exchange and the engine stands in zero context frames (conv / attention: the
    // receive slots are zeroed before use) or clip-local statistics (groupnorm).
    int ablate = VINF_ABLATE_NONE;
    void zero_recv_slots(const std::vector<vinf_xfer>& xs, cudaStream_t s) {
        for (const vinf_xfer& x : xs)
            if (!x.send) cuda_check(cudaMemsetAsync(ws + x.offset, 0, x.bytes, s), "ablation zero");
    }

    void stage_stub(uint32_t b, cudaStream_t s) { stub_frames(b, 0, L.f_clip, s); }
    void stub_frames(uint32_t b, uint32_t f0, uint32_t nf, cudaStream_t s);  // own frames [f0, f0+nf)
    void stage_conv(uint32_t b, cudaStream_t s);
    void stage_gn_apply(uint32_t b, cudaStream_t s);
    // W_vo = W_o W_v for block b (fuse_o), ahead of the GroupNorm fold that reads it (a fork
    // onto a second stream beside the stub measured the same step time: it stays inline)
    void launch_wvo(uint32_t b, cudaStream_t s);
    void stage_attention(uint32_t b, double t, cudaStream_t s);
    void stage_qkv(uint32_t b, cudaStream_t s);
    void project_qkv(uint32_t b, uint32_t frame0, uint32_t nframes, bool with_q, cudaStream_t s);
    int qkv_ready = -1;  // block whose own-frame Q/K/V projection has already run
    // bf16 mode: GroupNorm folded into the projections. The conv writes the raw GN input
    // straight into the attention buffer (so the exchanges ship raw frames), GN_APPLY
    // becomes one tiny kernel forming W' = W diag(s) and b' = W t, and the O GEMM adds the
    // residual as u * s + t. Needs the same (s, t) on every worker for every frame, and
    // zero receive/null frames to stay zero after projection, so not under GroupNorm or
    // attention ablation. VINF_NO_GN_FOLD=1 keeps the separate apply kernel.
    bool fold_env = [] {
        const char* v = getenv("VINF_NO_GN_FOLD");
        return !v || !*v || *v == '0';
    }();
    bool fold() const {
        return !f32() && fold_env && (ablate == VINF_ABLATE_NONE || ablate == VINF_ABLATE_CONV);
    }
    // One head: ctx W_o^T = P (X W_v^T) W_o^T = P (X (W_o W_v)^T), so the O projection is
    // absorbed into V (W_vo = W_o W_v, formed each step by a C^3 GEMM ahead of the GroupNorm
    // fold) and the attention core writes the block output (residual added in its epilogue).
    // VINF_NO_FUSE_O=1 keeps the separate O GEMM.
    bool fuse_o_env = [] {
        const char* v = getenv("VINF_NO_FUSE_O");
        return !v || !*v || *v == '0';
    }();
    bool fuse_o() const { return L.d.heads == 1 && fuse_o_env; }
    DevMat wfold_view() const {  // the folded Q/K/V weights (workspace), hi plane only
        DevMat m;
        m.rows = 3 * L.d.channels;
        m.K = L.d.channels;
        m.hi = at<__nv_bfloat16>(L.off_wfold);
        return m;
    }
    float* gn_aff() const { return at<float>(L.off_gnaff); }  // [s; t; b'(3C)]
};

void vinf_engine::stub_frames(uint32_t b, uint32_t f0, uint32_t nf, cudaStream_t s) {
    if (!nf) return;
    const EngineBlock& B = blocks.at(b);
    const uint64_t n = uint64_t(nf) * L.E, off = uint64_t(f0) * L.E;
    auto* u0 = at<__nv_bfloat16>(L.off_u0) + uint64_t(L.hc) * L.E + off;
    const void* x = static_cast<const uint8_t*>(x_of(b)) + off * (f32() ? 4 : 2);
    Span span(this, "stub", s);
    if (f32()) {
        auto* lo = at<__nv_bfloat16>(L.off_u0lo) + uint64_t(L.hc) * L.E + off;
        cuda_check(launch_stub(x, false, n, L.d.channels, B.stub_a(), B.stub_c(), at<float>(L.off_u0f) + off,
                               false, u0, lo, s),
                   "stub");
    } else {
        cuda_check(launch_stub(x, true, n, L.d.channels, B.stub_a(), B.stub_c(), u0, true, nullptr, nullptr, s),
                   "stub");
    }
    ++launches;
}

void vinf_engine::stage_conv(uint32_t b, cudaStream_t s) {
    const EngineBlock& B = blocks.at(b);
    const uint32_t C = L.d.channels;
    if (ablate == VINF_ABLATE_CONV) zero_recv_slots(L.xconv, s);
    Operand A;
    A.hi = at<__nv_bfloat16>(L.off_u0);
    A.lo = f32() ? at<__nv_bfloat16>(L.off_u0lo) : nullptr;
    A.rows = uint64_t(L.cf) * L.hw;
    A.cols = C;
    A.ld = C;
    std::vector<int64_t> ar, br;
    for (uint32_t j = 0; j < L.d.taps; ++j) {
        ar.push_back(int64_t(j) * L.hw);  // tap j reads own frame f at buffer frame f + j
        br.push_back(int64_t(j) * C);
    }
    Epilogue ep;
    // GroupNorm folding stores u1 - b (the bias is absorbed by the fold's shift, group_fold):
    // a smaller magnitude in bf16; the statistics are of u1 - b in either case
    ep.bias = fold() ? nullptr : B.conv_b();
    ep.res = f32() ? at(L.off_u0f) : static_cast<void*>(at<__nv_bfloat16>(L.off_u0) + uint64_t(L.hc) * L.E);
    ep.res_ld = C;
    ep.res_bf16 = !f32();
    ep.out = fold() ? static_cast<void*>(at<__nv_bfloat16>(L.off_u2) + uint64_t(L.ha) * L.E) : at(L.off_u1);
    ep.out_ld = C;
    ep.out_bf16 = !f32();
    // GroupNorm statistics of u1 fused into the GEMM epilogue: per-column (sum, sum of
    // squares) of the stored values, folded into per-group sums; workers all-reduce the
    // 2 * groups sums before GN_APPLY.
    const uint64_t rows = uint64_t(L.f_clip) * L.hw;
    float* colpart = at<float>(L.off_colstats);
    ep.colpart = colpart;
    {
        Span span(this, "conv_gemm", s);
        gemm(A, ar, B.conv, br, int64_t(rows), C, ep, f32(), s);
    }
    ++launches;
    Span span(this, "gn_stats", s);
    cuda_check(launch_colpart_to_groups(colpart, uint32_t(gemm_colpart_rows(int64_t(rows), int(C))), C, L.d.groups,
                                        B.conv_b(), double(rows), at<double>(L.off_sums),
                                        at<double>(L.off_scratch), s),
               "gn fold");
    launches += 1;
}

void vinf_engine::launch_wvo(uint32_t b, cudaStream_t s) {
    // V rows of W_qkv = W_o W_v (A = W_o [C x C], B = W_v^T)
    const EngineBlock& B = blocks.at(b);
    const uint32_t C = L.d.channels;
    Operand A;
    A.hi = B.wo.hi;
    A.lo = f32() ? B.wo.lo : nullptr;
    A.rows = C;
    A.cols = C;
    A.ld = C;
    Epilogue ep;
    ep.out = B.wqkv.hi + uint64_t(2) * C * C;
    ep.out_lo = f32() ? B.wqkv.lo + uint64_t(2) * C * C : nullptr;
    ep.out_ld = C;
    ep.out_bf16 = !f32();
    Span wspan(this, "wvo_gemm", s);
    gemm(A, {0}, B.wvT, {0}, C, C, ep, f32(), s);
    launches += 1;
}

void vinf_engine::stage_gn_apply(uint32_t b, cudaStream_t s) {
    const EngineBlock& B = blocks.at(b);
    double* sums = at<double>(L.off_sums);
    double* stats = at<double>(L.off_stats);
    const uint32_t G = L.d.groups;
    Span span(this, fold() ? "gn_fold" : "gn_apply", s);
    // mean = sum / n, var = sumsq / n - mean^2 over the whole video (n counts all clips),
    // formed by the apply kernel itself from the (all-reduced) sums
    (void)stats;
    auto* u2 = at<__nv_bfloat16>(L.off_u2) + uint64_t(L.ha) * L.E;
    if (fuse_o()) launch_wvo(b, s);
    if (fold()) {
        const uint32_t C = L.d.channels;
        float* aff = gn_aff();
        cuda_check(launch_group_fold(sums, gn_count(), C, G, B.gamma(), B.beta(), L.d.epsilon, B.wqkv.hi,
                                     3 * C, wfold_view().hi, aff + 2 * C, aff, B.conv_b(), s),
                   "gn fold");
    } else if (f32()) {
        auto* lo = at<__nv_bfloat16>(L.off_u2lo) + uint64_t(L.ha) * L.E;
        cuda_check(launch_group_apply(at(L.off_u1), false, uint64_t(L.f_clip) * L.hw,
                                      L.d.channels, G, sums, nullptr, B.gamma(), B.beta(),
                                      L.d.epsilon, at(L.off_u2f), false, u2, lo, s, gn_count()),
                   "gn apply");
    } else {
        cuda_check(launch_group_apply(at(L.off_u1), true, uint64_t(L.f_clip) * L.hw,
                                      L.d.channels, G, sums, nullptr, B.gamma(), B.beta(),
                                      L.d.epsilon, u2, true, nullptr, nullptr, s, gn_count()),
                   "gn apply");
    }
    launches += 1;
}

// Q/K/V (with_q) or K/V rows of `nframes` attention-buffer frames from frame0 on.
void vinf_engine::project_qkv(uint32_t b, uint32_t frame0, uint32_t nframes, bool with_q,
                              cudaStream_t s) {
    if (!nframes) return;
    const EngineBlock& B = blocks.at(b);
    const uint32_t C = L.d.channels;
    const uint64_t hw = L.hw;
    Operand A;
    A.hi = at<__nv_bfloat16>(L.off_u2);
    A.lo = f32() ? at<__nv_bfloat16>(L.off_u2lo) : nullptr;
    A.rows = uint64_t(L.af) * hw;
    A.cols = C;
    A.ld = C;
    // bf16 mode: one bf16 [af*HW, 3C] buffer; fp32 mode: the same as two bf16 planes (hi, lo)
    // written by the GEMM epilogue, the attention core's bf16x3 operands
    const uint64_t plane = uint64_t(L.af) * hw * 3 * C;
    auto* qkv = at<__nv_bfloat16>(L.off_qkv) + uint64_t(frame0) * hw * 3 * C + (with_q ? 0 : C);
    Epilogue ep;
    const bool fo = fold();
    if (fo) ep.bias = gn_aff() + 2 * C + (with_q ? 0 : C);
    ep.out = qkv;
    ep.out_lo = f32() ? qkv + plane : nullptr;
    ep.out_ld = 3 * C;
    ep.out_bf16 = !f32();
    Span span(this, with_q ? "qkv_gemm" : "kv_gemm_ctx", s);
    gemm(A, {int64_t(frame0) * int64_t(hw)}, fo ? wfold_view() : B.wqkv, {with_q ? 0 : int64_t(C)},
         int64_t(nframes) * int64_t(hw), with_q ? 3 * C : 2 * C, ep, f32(), s);
    ++launches;
}

// The own frames' Q/K/V projection only: it reads just this clip's normalised frames, so
// a driver may run it while the attention exchange is in flight (on another stream).
void vinf_engine::stage_qkv(uint32_t b, cudaStream_t s) {
    project_qkv(b, L.ha, L.f_clip, true, s);
    qkv_ready = int(b);
}

void vinf_engine::stage_attention(uint32_t b, double t, cudaStream_t s) {
    const EngineBlock& B = blocks.at(b);
    const uint32_t C = L.d.channels;
    const bool abl = ablate == VINF_ABLATE_ATTENTION;
    if (abl) zero_recv_slots(L.xattn, s);
    const uint64_t hw = L.hw;
    const bool bias_global = t > L.d.t_star;  // ops.cpp:298
    auto* ctx = at<__nv_bfloat16>(L.off_ctx);
    auto* ctxlo = f32() ? at<__nv_bfloat16>(L.off_ctxlo) : nullptr;
    const bool own_done = qkv_ready == int(b);
    qkv_ready = -1;
    {
        auto* qkv = at<__nv_bfloat16>(L.off_qkv);
        // own frames: Q, K, V (unless the QKV stage already ran for this block, overlapping
        // the attention exchange)
        if (!own_done) project_qkv(b, L.ha, L.f_clip, true, s);
        project_qkv(b, L.ha - L.npre_a, L.npre_a, false, s);  // pre halo: K, V
        // post halo, then the remote global frames (+ the zero null frame the ablated tables
        // point at): K, V; one launch when the post halo fills its slots (the two ranges are
        // then adjacent in the attention buffer)
        const uint32_t nrem = L.n_remote + (abl ? 1 : 0);
        if (L.npost_a == L.ha) {
            project_qkv(b, L.ha + L.f_clip, L.npost_a + nrem, false, s);
        } else {
            project_qkv(b, L.ha + L.f_clip, L.npost_a, false, s);
            project_qkv(b, 2 * L.ha + L.f_clip, nrem, false, s);
        }
        Span span(this, "attn_core", s);
        const uint64_t plane = uint64_t(L.af) * hw * 3 * C;
        FuseO fo;
        if (fuse_o()) {  // the block output straight from the core: ctx' + GN(u) (O GEMM epilogue below)
            fo.res = f32() ? at(L.off_u2f) : static_cast<void*>(at<__nv_bfloat16>(L.off_u2) + uint64_t(L.ha) * L.E);
            fo.res_bf16 = !f32();
            if (fold()) {
                fo.s = gn_aff();
                fo.t = gn_aff() + C;
            }
            fo.y = y_of(b);
            fo.y_bf16 = !f32();
        }
        cuda_check(launch_attention_core(qkv, f32() ? qkv + plane : nullptr, L.af, L.hw, C, L.d.heads, L.f_clip, L.ha,
                                         tt[(abl ? 2 : 0) + (bias_global ? 1 : 0)], L.scale, L.d.bias, ctx,
                                         ctxlo, s, &fo),
                   "attention core");
        ++launches;
    }
    if (fuse_o()) return;
    Operand O;
    O.hi = ctx;
    O.lo = ctxlo;
    O.rows = uint64_t(L.f_clip) * hw;
    O.cols = C;
    O.ld = C;
    Epilogue ep;
    ep.res = f32() ? at(L.off_u2f) : static_cast<void*>(at<__nv_bfloat16>(L.off_u2) + uint64_t(L.ha) * L.E);
    ep.res_ld = C;
    ep.res_bf16 = !f32();
    if (fold()) {  // the buffer holds the raw GN input: residual = GN(u) = u * s + t
        ep.res_scale = gn_aff();
        ep.bias = gn_aff() + C;
    }
    ep.out = y_of(b);
    ep.out_ld = C;
    ep.out_bf16 = !f32();
    Span span(this, "o_gemm", s);
    gemm(O, {0}, B.wo, {0}, int64_t(L.f_clip) * hw, C, ep, f32(), s);
    ++launches;
}


// ---- clip-parallel executor ----------------------------------------------------------

void vinf_engine::dist_init() {
    if (dist.cs) return;
    int lo = 0, hi = 0;
    cuda_check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "stream priorities");
    // the exchanges' copy / NCCL kernels are scheduled ahead of queued compute blocks
    cuda_check(cudaStreamCreateWithPriority(&dist.cs, cudaStreamNonBlocking, hi), "comm stream");
    for (auto& e : dist.ev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    dist.xconv = matching_order(L.xconv);
    dist.xattn = matching_order(L.xattn);
}

// One block of eps_theta_worker (pipeline.cpp:150-170) with the paper's 3-step sync:
//  1. conv halo: the clip's boundary frames are stubbed first and shipped on the comm
//     stream while the interior frames are stubbed (sync_contexts T2/T3,
//     clip_parallel.cpp:160-188, minus the even/odd staging NVSwitch does not need);
//  2. GroupNorm: one all-reduce of the 2*groups (sum, sum of squares) partials on the
//     compute stream (the reference's two all-gather rounds, clip_parallel.cpp:242-253);
//  3. attention context: halo frames + the sampled global frames each receiver lacks
//     (T1, clip_parallel.cpp:114-148) on the comm stream while the own frames are
//     projected to Q/K/V; their K/V projection and the attention core wait for it.
// Every comm-stream operation starts after an event of the compute stream and the
// compute stream waits for it before the receive slots are read, so all communicator
// operations of a worker are ordered in time (one communicator serves both streams).
void vinf_engine::dist_block(uint32_t b, double t, vinf_comm* comm, cudaStream_t s) {
    const bool multi = comm->nranks > 1;
    cudaStream_t cs = dist.cs;
    const bool x_conv = multi && ablate != VINF_ABLATE_CONV && !dist.xconv.empty();
    if (x_conv) {
        const uint32_t h = L.hc, fc = L.f_clip;
        const bool split = 2 * h < fc;
        if (split) {
            stub_frames(b, 0, h, s);
            stub_frames(b, fc - h, h, s);
        } else {
            stage_stub(b, s);
        }
        cuda_check(cudaEventRecord(dist.ev[0], s), "event");
        cuda_check(cudaStreamWaitEvent(cs, dist.ev[0], 0), "wait");
        {
            Span span(this, "xchg_conv", cs);
            run_exchange(comm, dist.xconv, ws, cs);
        }
        cuda_check(cudaEventRecord(dist.ev[1], cs), "event");
        if (split) stub_frames(b, h, fc - 2 * h, s);
        cuda_check(cudaStreamWaitEvent(s, dist.ev[1], 0), "wait");
    } else {
        stage_stub(b, s);
    }
    stage_conv(b, s);
    if (multi && ablate != VINF_ABLATE_GROUPNORM) {
        Span span(this, "allreduce_gn", s);
        comm->allreduce_sum_f64(at<double>(L.off_sums), 2ull * L.d.groups, s);
    }
    const bool x_attn = multi && ablate != VINF_ABLATE_ATTENTION && !dist.xattn.empty();
    auto start_attn = [&] {
        cuda_check(cudaEventRecord(dist.ev[2], s), "event");
        cuda_check(cudaStreamWaitEvent(cs, dist.ev[2], 0), "wait");
        Span span(this, "xchg_attn", cs);
        run_exchange(comm, dist.xattn, ws, cs);
        cuda_check(cudaEventRecord(dist.ev[3], cs), "event");
    };
    // GroupNorm folded (bf16): the conv already wrote the raw frames the exchange ships,
    // so it overlaps the fold as well; otherwise it ships the normalised frames
    if (x_attn && fold()) start_attn();
    stage_gn_apply(b, s);
    if (x_attn && !fold()) start_attn();
    if (x_attn) {
        stage_qkv(b, s);
        cuda_check(cudaStreamWaitEvent(s, dist.ev[3], 0), "wait");
    }
    stage_attention(b, t, s);
}

namespace {

void dist_stack(vinf_engine* e, double t, vinf_comm* comm, cudaStream_t s) {
    for (uint32_t b = 0; b < e->blocks.size(); ++b) e->dist_block(b, t, comm, s);
}

// NCCL operations are graph-capturable: the stack of each timestep regime is captured
// once (after one eager pass) and replayed, like the single-worker path.
void forward_dist(vinf_engine* e, double t, vinf_comm* comm, bool use_graph, cudaStream_t s) {
    e->dist_init();
    if (!use_graph || e->profiling || !comm->capturable() || !e->use_graphs) {
        dist_stack(e, t, comm, s);
        return;
    }
    if (e->dist.graph_comm != comm) {
        e->drop_graphs();
        e->dist.graph_comm = comm;
    }
    auto& g = e->dist.graphs[t > e->L.d.t_star ? 1 : 0];
    if (!g.exec && g.calls++ >= 1) {
        if (!e->cap_stream)
            cuda_check(cudaStreamCreateWithFlags(&e->cap_stream, cudaStreamNonBlocking), "capture stream");
        const uint64_t l0 = e->launches;
        const uint64_t b0 = comm->bytes_sent, m0 = comm->messages_sent;
        cuda_check(cudaStreamBeginCapture(e->cap_stream, cudaStreamCaptureModeThreadLocal), "begin capture");
        try {
            dist_stack(e, t, comm, e->cap_stream);
        } catch (...) {
            cudaGraph_t broken = nullptr;
            cudaStreamEndCapture(e->cap_stream, &broken);
            if (broken) cudaGraphDestroy(broken);
            e->launches = l0;
            throw;
        }
        cudaGraph_t graph = nullptr;
        cuda_check(cudaStreamEndCapture(e->cap_stream, &graph), "end capture");
        const cudaError_t ie = cudaGraphInstantiate(&g.exec, graph, 0);
        cudaGraphDestroy(graph);
        cuda_check(ie, "graph instantiate");
        g.nlaunch = e->launches - l0;
        g.nbytes = comm->bytes_sent - b0;
        g.nmsgs = comm->messages_sent - m0;
        e->launches = l0;
        comm->bytes_sent = b0;
        comm->messages_sent = m0;
    }
    if (g.exec) {
        cuda_check(cudaGraphLaunch(g.exec, s), "graph launch");
        e->launches += g.nlaunch;
        comm->bytes_sent += g.nbytes;
        comm->messages_sent += g.nmsgs;
    } else {
        dist_stack(e, t, comm, s);
    }
}

void check_comm(const vinf_engine* e, const vinf_comm* comm) {
    if (!comm) shape_error("null communicator");
    if (comm->nranks != e->L.d.workers || comm->rank != e->L.d.worker)
        config_error("communicator rank " + std::to_string(comm->rank) + " of " + std::to_string(comm->nranks) +
                     " does not match the engine's worker " + std::to_string(e->L.d.worker) + " of " +
                     std::to_string(e->L.d.workers));
}

}  // namespace

// ---- C ABI (engine part) ---------------------------------------------------------

namespace vinf {
int guarded_call(const std::function<void()>& f);
}

extern "C" {

int vinf_engine_create(const vinf_layout* l, void* workspace, void* stream, vinf_engine** out) {
    return guarded_call([&] {
        if (!l || !out) shape_error("null argument");
        if (!workspace) shape_error("null workspace");
        auto s = static_cast<cudaStream_t>(stream);
        auto* e = new vinf_engine(l->L);
        e->ws = static_cast<uint8_t*>(workspace);
        const Layout& L = e->L;
        cuda_check(cudaMemsetAsync(e->ws, 0, L.total, s), "workspace memset");
        std::vector<uint8_t> blob[4];
        for (int b = 0; b < 4; ++b) {
            uint8_t* p = e->at(L.off_tok[b]);
            blob[b].resize(L.tok[b].blob_bytes());
            L.tok[b].pack(blob[b].data());
            cuda_check(cudaMemcpyAsync(p, blob[b].data(), blob[b].size(), cudaMemcpyHostToDevice, s),
                       "tokens");
            e->tt[b] = L.tok[b].view(p);
        }
        const uint32_t C = L.d.channels;
        e->blocks.resize(L.d.blocks);
        for (auto& B : e->blocks) {
            B.C = C;
            cuda_check(cudaMalloc(&B.f32, sizeof(float) * 5 * C), "cudaMalloc(block)");
            B.conv.alloc(L.d.taps * C, C);
            B.wqkv.alloc(3 * C, C);
            B.wo.alloc(C, C);
            B.wvT.alloc(C, C);
        }
        cuda_check(cudaStreamSynchronize(s), "engine create sync");
        *out = e;
    });
}

void vinf_engine_destroy(vinf_engine* e) {
    if (!e) return;
    e->drop_graphs();
    if (e->cap_stream) cudaStreamDestroy(e->cap_stream);
    if (e->dist.cs) cudaStreamDestroy(e->dist.cs);
    for (cudaEvent_t ev : e->dist.ev)
        if (ev) cudaEventDestroy(ev);
    for (cudaEvent_t ev : e->pool) cudaEventDestroy(ev);
    for (auto& B : e->blocks) {
        if (B.f32) cudaFree(B.f32);
        B.conv.release();
        B.wqkv.release();
        B.wo.release();
        B.wvT.release();
    }
    delete e;
}

int vinf_engine_set_block(vinf_engine* e, uint32_t block, const float* stub_a,
                          const float* stub_c, const float* conv_w, const float* conv_b,
                          const float* gamma, const float* beta, const float* wq, const float* wk,
                          const float* wv, const float* wo, void* stream) {
    return guarded_call([&] {
        if (e) e->drop_graphs();
        if (!e) shape_error("null engine");
        if (block >= e->blocks.size()) range_error("block index out of range");
        auto s = static_cast<cudaStream_t>(stream);
        EngineBlock& B = e->blocks[block];
        const uint32_t C = B.C;
        const size_t vb = sizeof(float) * C;
        const float* vecs[5] = {stub_a, stub_c, conv_b, gamma, beta};
        for (int i = 0; i < 5; ++i) {
            if (!vecs[i]) shape_error("null block parameter");
            cuda_check(cudaMemcpyAsync(B.f32 + i * C, vecs[i], vb, cudaMemcpyDeviceToDevice, s), "params");
        }
        if (!conv_w || !wq || !wk || !wv || !wo) shape_error("null block weight");
        B.conv.from_f32(conv_w, s);
        const size_t mat = size_t(C) * C;
        float* tmp = nullptr;
        cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&tmp), 3 * mat * 4, s), "tmp");
        cuda_check(cudaMemcpyAsync(tmp, wq, mat * 4, cudaMemcpyDeviceToDevice, s), "wq");
        cuda_check(cudaMemcpyAsync(tmp + mat, wk, mat * 4, cudaMemcpyDeviceToDevice, s), "wk");
        cuda_check(cudaMemcpyAsync(tmp + 2 * mat, wv, mat * 4, cudaMemcpyDeviceToDevice, s), "wv");
        B.wqkv.from_f32(tmp, s);
        cuda_check(launch_transpose_f32(wv, tmp, C, C, s), "transpose W_v");
        B.wvT.from_f32(tmp, s);
        cuda_check(cudaFreeAsync(tmp, s), "tmp");
        B.wo.from_f32(wo, s);
    });
}

int vinf_engine_init_weights(vinf_engine* e, uint64_t weight_seed, void* stream) {
    return guarded_call([&] {
        if (!e) shape_error("null engine");
        e->drop_graphs();
        auto s = static_cast<cudaStream_t>(stream);
        const uint32_t C = e->L.d.channels, taps = e->L.d.taps;
        const float mat = 1.0f / std::sqrt(float(C));  // pipeline.cpp:44
        const size_t m = size_t(C) * C;
        float* tmp = nullptr;
        const size_t n_tmp = size_t(taps) * m + 4 * m + 5 * C;
        cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&tmp), n_tmp * 4, s), "tmp");
        float* cw = tmp;
        float* wq = cw + size_t(taps) * m;
        float* wk = wq + m;
        float* wv = wk + m;
        float* wo = wv + m;
        float* vec = wo + m;  // stub_a, stub_c, conv_b, gamma, beta
        for (uint32_t b = 0; b < e->blocks.size(); ++b) {
            auto salt = [&](uint64_t slot) { return mix_seed(weight_seed, uint64_t(b) * 16 + slot); };
            // spatial_stub_coeffs (ops.cpp:57-65): a = draws [0, C), c = draws [C, 2C)
            cuda_check(launch_fill_seeded(vec, false, C, salt(kStub), 0, 1.0f, s), "fill");
            cuda_check(launch_fill_seeded(vec + C, false, C, salt(kStub), C, 1.0f, s), "fill");
            cuda_check(launch_fill_seeded(cw, false, uint64_t(taps) * m, salt(kConvW), 0, mat, s), "fill");
            cuda_check(launch_fill_seeded(vec + 2 * C, false, C, salt(kConvB), 0, 1.0f, s), "fill");
            cuda_check(launch_fill_seeded(vec + 3 * C, false, C, salt(kGamma), 0, 1.0f, s), "fill");
            cuda_check(launch_fill_seeded(vec + 4 * C, false, C, salt(kBeta), 0, 1.0f, s), "fill");
            cuda_check(launch_fill_seeded(wq, false, m, salt(kWq), 0, mat, s), "fill");
            cuda_check(launch_fill_seeded(wk, false, m, salt(kWk), 0, mat, s), "fill");
            cuda_check(launch_fill_seeded(wv, false, m, salt(kWv), 0, mat, s), "fill");
            cuda_check(launch_fill_seeded(wo, false, m, salt(kWo), 0, mat, s), "fill");
            const int rc = vinf_engine_set_block(e, b, vec, vec + C, cw, vec + 2 * C, vec + 3 * C,
                                                 vec + 4 * C, wq, wk, wv, wo, stream);
            if (rc) throw Error(rc, vinf_last_error());
        }
        cuda_check(cudaFreeAsync(tmp, s), "tmp");
        cuda_check(cudaStreamSynchronize(s), "init weights sync");
    });
}

int vinf_engine_stage(vinf_engine* e, uint32_t block, int stage, double t, void* stream) {
    return guarded_call([&] {
        if (!e) shape_error("null engine");
        if (block >= e->blocks.size()) range_error("block index out of range");
        auto s = static_cast<cudaStream_t>(stream);
        switch (stage) {
            case VINF_STAGE_STUB: e->stage_stub(block, s); break;
            case VINF_STAGE_CONV: e->stage_conv(block, s); break;
            case VINF_STAGE_GN_APPLY: e->stage_gn_apply(block, s); break;
            case VINF_STAGE_ATTENTION: e->stage_attention(block, t, s); break;
            case VINF_STAGE_QKV: e->stage_qkv(block, s); break;
            default: range_error("unknown stage");
        }
    });
}

namespace {

void run_stack(vinf_engine* e, double t, cudaStream_t s) {
    for (uint32_t b = 0; b < e->blocks.size(); ++b) {
        e->stage_stub(b, s);
        e->stage_conv(b, s);
        e->stage_gn_apply(b, s);
        e->stage_attention(b, t, s);
    }
}

// One pass of the block stack: replayed from the regime's graph once it has been seen
// twice (the first pass runs eagerly and sets every lazily-initialised kernel attribute).
void forward_stack(vinf_engine* e, double t, cudaStream_t s) {
    if (e->profiling || !e->use_graphs) {
        run_stack(e, t, s);
        return;
    }
    auto& g = e->graphs[t > e->L.d.t_star ? 1 : 0];
    if (!g.exec && g.calls++ >= 1) {
        if (!e->cap_stream)
            cuda_check(cudaStreamCreateWithFlags(&e->cap_stream, cudaStreamNonBlocking), "capture stream");
        const uint64_t l0 = e->launches;
        cuda_check(cudaStreamBeginCapture(e->cap_stream, cudaStreamCaptureModeThreadLocal), "begin capture");
        try {
            run_stack(e, t, e->cap_stream);
        } catch (...) {
            cudaGraph_t broken = nullptr;
            cudaStreamEndCapture(e->cap_stream, &broken);
            if (broken) cudaGraphDestroy(broken);
            e->launches = l0;
            throw;
        }
        cudaGraph_t graph = nullptr;
        cuda_check(cudaStreamEndCapture(e->cap_stream, &graph), "end capture");
        const cudaError_t ie = cudaGraphInstantiate(&g.exec, graph, 0);
        cudaGraphDestroy(graph);
        cuda_check(ie, "graph instantiate");
        g.nlaunch = e->launches - l0;
        e->launches = l0;
    }
    if (g.exec) {
        cuda_check(cudaGraphLaunch(g.exec, s), "graph launch");
        e->launches += g.nlaunch;
    } else {
        run_stack(e, t, s);
    }
}

}  // namespace

int vinf_engine_forward(vinf_engine* e, double t, void* stream) {
    return guarded_call([&] {
        if (!e) shape_error("null engine");
        if (e->L.d.workers != 1)
            config_error("vinf_engine_forward runs a single worker; use vinf_engine_stage with a "
                         "transport for workers > 1");
        forward_stack(e, t, static_cast<cudaStream_t>(stream));
    });
}

int vinf_engine_set_ablation(vinf_engine* e, int kind) {
    return guarded_call([&] {
        if (!e) shape_error("null engine");
        if (kind < VINF_ABLATE_NONE || kind > VINF_ABLATE_ATTENTION)
            config_error("ablation kind must be none, conv, groupnorm or attention");
        e->ablate = kind;
        e->drop_graphs();
    });
}

int vinf_engine_euler(vinf_engine* e, double lambda, void* stream) {
    return guarded_call([&] {
        if (!e) shape_error("null engine");
        auto s = static_cast<cudaStream_t>(stream);
        vinf_engine::Span span(e, "euler", s);
        cuda_check(launch_euler(e->at(e->L.off_x), e->at(e->L.off_y), !e->f32(), e->clip_elems(),
                                lambda, s),
                   "euler");
        e->launches += 1;
    });
}

int vinf_engine_denoise(vinf_engine* e, uint32_t steps, void* stream) {
    return guarded_call([&] {
        if (!e) shape_error("null engine");
        if (steps == 0) config_error("denoising needs at least one step");
        if (e->L.d.workers != 1)
            config_error("vinf_engine_denoise runs a single worker; use the staged loop for workers > 1");
        auto s = static_cast<cudaStream_t>(stream);
        // worker_denoise (pipeline.cpp:174-191): t_j = 1000 j / steps, j = steps..1
        for (uint32_t j = steps; j >= 1; --j) {
            const double t = 1000.0 * j / steps;
            forward_stack(e, t, s);
            cuda_check(launch_euler(e->at(e->L.off_x), e->at(e->L.off_y), !e->f32(),
                                    e->clip_elems(), 1.0 / steps, s),
                       "euler");
            e->launches += 1;
        }
    });
}

int vinf_engine_io(const vinf_engine* e, void** x, void** y) {
    return guarded_call([&] {
        if (!e) shape_error("null engine");
        if (x) *x = e->at(e->L.off_x);
        if (y) *y = e->at(e->L.off_y);
    });
}

uint64_t vinf_engine_launches(const vinf_engine* e) { return e ? e->launches : 0; }

int vinf_engine_profile(vinf_engine* e, int enable) {
    return guarded_call([&] {
        if (!e) shape_error("null engine");
        e->profiling = enable != 0;
        e->recs.clear();
        e->pool_used = 0;
    });
}

int vinf_engine_kernel_stats(vinf_engine* e, char* names, uint32_t name_cap, double* total_ms,
                             uint64_t* counts, uint32_t cap, uint32_t* n_out) {
    return guarded_call([&] {
        if (!e) shape_error("null engine");
        std::vector<std::string> keys;
        std::vector<double> ms;
        std::vector<uint64_t> cnt;
        for (const auto& r : e->recs) {
            cuda_check(cudaEventSynchronize(r.b), "event sync");
            float t = 0.f;
            cuda_check(cudaEventElapsedTime(&t, r.a, r.b), "event elapsed");
            size_t k = 0;
            while (k < keys.size() && keys[k] != r.name) ++k;
            if (k == keys.size()) {
                keys.push_back(r.name);
                ms.push_back(0.0);
                cnt.push_back(0);
            }
            ms[k] += t;
            cnt[k] += 1;
        }
        if (n_out) *n_out = uint32_t(keys.size());
        std::string joined;
        for (size_t k = 0; k < keys.size(); ++k) joined += (k ? "," : "") + keys[k];
        if (names && name_cap) {
            std::strncpy(names, joined.c_str(), name_cap - 1);
            names[name_cap - 1] = 0;
        }
        for (size_t k = 0; k < keys.size() && k < cap; ++k) {
            if (total_ms) total_ms[k] = ms[k];
            if (counts) counts[k] = cnt[k];
        }
        e->recs.clear();
        e->pool_used = 0;
    });
}

int vinf_layout_run_exchange(const vinf_layout* l, int stage, void* base, vinf_comm* comm, void* stream) {
    return guarded_call([&] {
        if (!l || !comm) shape_error("null argument");
        if (!base) shape_error("null workspace");
        if (stage != VINF_XCHG_CONV && stage != VINF_XCHG_ATTN) range_error("unknown exchange stage");
        if (comm->nranks != l->L.d.workers || comm->rank != l->L.d.worker)
            config_error("communicator rank does not match the layout's worker");
        run_exchange(comm, matching_order(stage == VINF_XCHG_CONV ? l->L.xconv : l->L.xattn),
                     static_cast<uint8_t*>(base), static_cast<cudaStream_t>(stream));
    });
}

int vinf_engine_exchange(vinf_engine* e, int stage, vinf_comm* comm, void* stream) {
    return guarded_call([&] {
        if (!e) shape_error("null engine");
        check_comm(e, comm);
        if (stage != VINF_XCHG_CONV && stage != VINF_XCHG_ATTN) range_error("unknown exchange stage");
        e->dist_init();
        auto s = static_cast<cudaStream_t>(stream);
        vinf_engine::Span span(e, stage == VINF_XCHG_CONV ? "xchg_conv" : "xchg_attn", s);
        run_exchange(comm, stage == VINF_XCHG_CONV ? e->dist.xconv : e->dist.xattn, e->ws, s);
    });
}

int vinf_engine_allreduce_sums(vinf_engine* e, vinf_comm* comm, void* stream) {
    return guarded_call([&] {
        if (!e) shape_error("null engine");
        check_comm(e, comm);
        auto s = static_cast<cudaStream_t>(stream);
        vinf_engine::Span span(e, "allreduce_gn", s);
        comm->allreduce_sum_f64(e->at<double>(e->L.off_sums), 2ull * e->L.d.groups, s);
    });
}

int vinf_engine_forward_dist(vinf_engine* e, double t, vinf_comm* comm, int use_graph, void* stream) {
    return guarded_call([&] {
        if (!e) shape_error("null engine");
        check_comm(e, comm);
        forward_dist(e, t, comm, use_graph != 0, static_cast<cudaStream_t>(stream));
    });
}

int vinf_engine_denoise_dist(vinf_engine* e, uint32_t steps, vinf_comm* comm, int use_graph, void* stream) {
    return guarded_call([&] {
        if (!e) shape_error("null engine");
        check_comm(e, comm);
        if (steps == 0) config_error("denoising needs at least one step");
        auto s = static_cast<cudaStream_t>(stream);
        for (uint32_t j = steps; j >= 1; --j) {  // timestep_grid (pipeline.cpp:75-81)
            const double t = 1000.0 * j / steps;
            forward_dist(e, t, comm, use_graph != 0, s);
            cuda_check(launch_euler(e->at(e->L.off_x), e->at(e->L.off_y), !e->f32(), e->clip_elems(), 1.0 / steps, s),
                       "euler");
            e->launches += 1;
        }
    });
}

}  // extern "C"
