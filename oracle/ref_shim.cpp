// extern "C" shim over the UNMODIFIED reference library — TEST / BASELINE INFRASTRUCTURE ONLY.
//
// oracle/Makefile compiles this file together with the reference sources where
// they lie (/root/reference/proj/src/core/*.cpp; nothing is copied) into
// oracle/_ref/libvinf_ref.so. tests/ use it to pin oracle/vinf_oracle.c and to
// generate tests/golden/; bench.py uses ref_execute_run as the reference CPU arm
// (execute_run, runner.cpp:213-227 — the reference's own public run path).
#include <chrono>
#include <cstring>
#include <exception>
#include <vector>

#include "core/clip_parallel.hpp"
#include "core/config.hpp"
#include "core/ops.hpp"
#include "core/pipeline.hpp"
#include "core/runner.hpp"
#include "core/tensor.hpp"
#include "core/transport_inproc.hpp"

using namespace vinf;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 1;
    } catch (const RangeError& e) {
        g_err = e.what();
        return 2;
    } catch (const ShapeError& e) {
        g_err = e.what();
        return 3;
    } catch (const ProtocolError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

Tensor wrap(const float* p, uint32_t f, uint32_t h, uint32_t w, uint32_t c) {
    Dims d{f, h, w, c};
    return Tensor(d, std::vector<float>(p, p + d.total()));
}

void unwrap(const Tensor& t, float* out) { std::memcpy(out, t.data(), t.size() * sizeof(float)); }

AttentionParams attn_params(uint32_t C, const float* wq, const float* wk, const float* wv,
                            const float* wo, float scale) {
    AttentionParams p;
    p.dim = C;
    p.scale = scale;
    const size_t n = size_t(C) * C;
    p.wq.assign(wq, wq + n);
    p.wk.assign(wk, wk + n);
    p.wv.assign(wv, wv + n);
    p.wo.assign(wo, wo + n);
    return p;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_fill_seeded(float* out, uint64_t n, uint64_t seed, uint64_t first_elem) {
    return guarded([&] {
        unwrap(tensor_from_seed_at(Dims{1, 1, 1, uint32_t(n)}, seed, first_elem), out);
    });
}

int ref_build_block(uint32_t C, uint32_t taps, uint32_t groups, uint64_t weight_seed,
                    uint32_t blocks, uint32_t block, float* stub_a, float* stub_c, float* conv_w,
                    float* conv_b, float* gamma, float* beta, float* wq, float* wk, float* wv,
                    float* wo) {
    return guarded([&] {
        ModelConfig mc;
        mc.blocks = blocks;
        mc.channels = C;
        mc.taps = taps;
        mc.groups = groups;
        mc.weight_seed = weight_seed;
        const Model m = build_model(mc);
        const Block& b = m.blocks.at(block);
        auto cp = [](const std::vector<float>& v, float* o) {
            std::memcpy(o, v.data(), v.size() * sizeof(float));
        };
        cp(b.stub_a, stub_a); cp(b.stub_c, stub_c);
        cp(b.conv.weights, conv_w); cp(b.conv.bias, conv_b);
        cp(b.norm.gamma, gamma); cp(b.norm.beta, beta);
        cp(b.attn.wq, wq); cp(b.attn.wk, wk); cp(b.attn.wv, wv); cp(b.attn.wo, wo);
    });
}

int ref_conv_over_extended(const float* ext, uint32_t ext_f, uint32_t H, uint32_t W, uint32_t C,
                           uint32_t out_start, uint32_t out_len, uint32_t taps, const float* wts,
                           const float* bias, float* out) {
    return guarded([&] {
        ConvKernel k;
        k.taps = taps;
        k.weights.assign(wts, wts + size_t(taps) * C * C);
        k.bias.assign(bias, bias + C);
        unwrap(conv_over_extended(wrap(ext, ext_f, H, W, C), out_start, out_len, k), out);
    });
}

int ref_group_norm(const float* v, uint32_t F, uint32_t H, uint32_t W, uint32_t C, uint32_t groups,
                   const float* gamma, const float* beta, float eps, float* out, double* means,
                   double* vars) {
    return guarded([&] {
        GroupNormParams p;
        p.groups = groups;
        p.gamma.assign(gamma, gamma + C);
        p.beta.assign(beta, beta + C);
        p.epsilon = eps;
        const Tensor x = wrap(v, F, H, W, C);
        unwrap(group_norm(x, p), out);
        if (means || vars) {
            const auto m = group_means(x, groups);
            const auto s = group_sqdev(x, groups, m);
            if (means) std::memcpy(means, m.data(), groups * sizeof(double));
            if (vars) std::memcpy(vars, s.data(), groups * sizeof(double));
        }
    });
}

int ref_dual_scope(const float* v, uint32_t F, uint32_t H, uint32_t W, uint32_t C, double t,
                   const float* wq, const float* wk, const float* wv, const float* wo, float scale,
                   uint32_t n_local, uint32_t n_global, float bias, double t_star, float* out,
                   uint64_t* counters) {
    return guarded([&] {
        DualScopeConfig cfg;
        cfg.n_local = n_local;
        cfg.n_global = n_global;
        cfg.bias = bias;
        cfg.t_star = t_star;
        AttnCounters c;
        unwrap(dual_scope_reference(wrap(v, F, H, W, C), t, attn_params(C, wq, wk, wv, wo, scale),
                                    cfg, &c),
               out);
        if (counters) {
            counters[0] = c.score_entries;
            counters[1] = c.queries;
            counters[2] = c.max_tokens_per_query;
        }
    });
}

int ref_attention_full(const float* v, uint32_t F, uint32_t H, uint32_t W, uint32_t C,
                       const float* wq, const float* wk, const float* wv, const float* wo,
                       float scale, float* out, double* row_sums) {
    return guarded([&] {
        ScoreProbe probe;
        unwrap(attention_full(wrap(v, F, H, W, C), attn_params(C, wq, wk, wv, wo, scale),
                              row_sums ? &probe : nullptr),
               out);
        if (row_sums) std::memcpy(row_sums, probe.row_sums.data(), probe.row_sums.size() * 8);
    });
}

int ref_build_local_window(uint32_t a, uint32_t frames, uint32_t n_local, uint32_t* out) {
    int n = -1;
    const int rc = guarded([&] {
        const auto w = build_local_window(a, frames, n_local);
        std::memcpy(out, w.data(), w.size() * 4);
        n = int(w.size());
    });
    return rc ? -1 : n;
}

int ref_build_global_index_set(uint32_t frames, uint32_t n_global, uint32_t* out) {
    int n = -1;
    const int rc = guarded([&] {
        const auto g = build_global_index_set(frames, n_global);
        std::memcpy(out, g.data(), g.size() * 4);
        n = int(g.size());
    });
    return rc ? -1 : n;
}

int ref_global_members_in_range(uint32_t frames, uint32_t n_global, uint32_t start, uint32_t len,
                                uint32_t* out) {
    int n = -1;
    const int rc = guarded([&] {
        const auto g = global_members_in_range(frames, n_global, FrameRange{start, len});
        std::memcpy(out, g.data(), g.size() * 4);
        n = int(g.size());
    });
    return rc ? -1 : n;
}

int ref_predict_sync_traffic(uint32_t frames, uint32_t workers, uint32_t halo,
                             uint32_t global_frames, uint32_t worker, uint64_t frame_bytes,
                             uint64_t* out) {
    return guarded([&] {
        const ClipPlan plan = make_plan(frames, workers);
        const LayerHaloSpec spec{LayerKind::Attention, halo, global_frames};
        const auto p = predict_sync_traffic(plan, spec, worker, frame_bytes);
        out[0] = p.bytes_sent;
        out[1] = p.bytes_contributed;
        out[2] = p.messages;
    });
}

int ref_predict_groupnorm_traffic(uint32_t frames, uint32_t workers, uint32_t groups,
                                  uint32_t worker, uint64_t* out) {
    return guarded([&] {
        const auto p = predict_groupnorm_traffic(make_plan(frames, workers), groups, worker);
        out[0] = p.bytes_sent;
        out[1] = p.bytes_contributed;
        out[2] = p.messages;
    });
}

// One block (stub -> conv+res -> GN -> dual-scope attn+res) at timestep t over the
// whole video, either sequentially (workers == 0: eps_theta_sequential,
// pipeline.cpp:102-111) or clip-parallel over `workers` in-process threads
// (eps_theta_worker, pipeline.cpp:145-172). Weights come from build_model.
// Measured TRANSPORT bytes per worker (optional, [workers][3] for conv/gn/attn)
// let tests check the traffic closed forms.
int ref_block_forward(const float* x, uint32_t F, uint32_t H, uint32_t W, uint32_t C,
                      uint32_t taps, uint32_t groups, uint64_t weight_seed, uint32_t n_local,
                      uint32_t n_global, float bias, double t_star, double t, uint32_t workers,
                      float* out, uint64_t* bytes_per_kind) {
    return guarded([&] {
        ModelConfig mc;
        mc.blocks = 1;
        mc.channels = C;
        mc.taps = taps;
        mc.groups = groups;
        mc.weight_seed = weight_seed;
        mc.dual_scope.n_local = n_local;
        mc.dual_scope.n_global = n_global;
        mc.dual_scope.bias = bias;
        mc.dual_scope.t_star = t_star;
        const Model m = build_model(mc);
        const Tensor full = wrap(x, F, H, W, C);
        if (workers == 0) {
            unwrap(eps_theta_sequential(full, t, m), out);
            return;
        }
        const ClipPlan plan = make_plan(F, workers);
        check_halo_constraints(mc, plan.f_clip);
        const auto clips = partition(full, workers);
        std::vector<Tensor> res(workers);
        std::vector<WorkerMetrics> wm(workers);
        run_inproc_workers(workers, false, [&](Transport& tr) {
            uint32_t call = 1;
            res[tr.rank()] = eps_theta_worker(tr, plan, clips[tr.rank()], t, m, &call,
                                              &wm[tr.rank()]);
        });
        unwrap(concat_frames(res), out);
        if (bytes_per_kind) {
            for (uint32_t i = 0; i < workers; ++i) {
                bytes_per_kind[3 * i + 0] = wm[i].conv.bytes_sent;
                bytes_per_kind[3 * i + 1] = wm[i].groupnorm.bytes_sent;
                bytes_per_kind[3 * i + 2] = wm[i].attention.bytes_sent;
            }
        }
    });
}

// The reference's public run path (execute_run, runner.cpp:213-227), used as the
// CPU baseline: workers == 0 forces the sequential oracle, else in-process
// clip-parallel threads. Returns wall seconds as measured around the call.
int ref_execute_run(uint32_t F, uint32_t H, uint32_t W, uint32_t C, uint32_t groups,
                    uint32_t n_local, uint32_t n_global, uint32_t blocks, uint32_t steps,
                    uint32_t workers, uint64_t seed, uint64_t weight_seed, float* x0_out,
                    double* wall_seconds) {
    return guarded([&] {
        RunConfig cfg;
        cfg.frames = F;
        cfg.height = H;
        cfg.width = W;
        cfg.channels = C;
        cfg.groups = groups;
        cfg.n_local = n_local;
        cfg.n_global = n_global;
        cfg.blocks = blocks;
        cfg.steps = steps;
        cfg.seed = seed;
        cfg.weight_seed = weight_seed;
        cfg.sequential = workers == 0;
        cfg.workers = workers == 0 ? 1 : workers;
        const auto t0 = std::chrono::steady_clock::now();
        RunResult r = execute_run(cfg);
        const double dt =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (wall_seconds) *wall_seconds = dt;
        if (x0_out) unwrap(r.x0, x0_out);
    });
}

}  // extern "C"
