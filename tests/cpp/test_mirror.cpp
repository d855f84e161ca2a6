// C++ parity test through the header-only mirror (include/vinf_temporal.hpp) of the
// reference API: device results vs the CPU oracle (oracle/vinf_oracle.c), plus the
// reference error taxonomy. Built and run by tests/test_cpp_mirror.py.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <vector>

#include "vinf_oracle.h"
#include "vinf_temporal.hpp"

namespace b = vinf::b200;

static double normwise(const std::vector<float>& got, const std::vector<float>& want) {
    double md = 0, mr = 0;
    for (size_t i = 0; i < got.size(); ++i) {
        md = std::fmax(md, std::fabs(double(got[i]) - double(want[i])));
        mr = std::fmax(mr, std::fabs(double(want[i])));
    }
    return md / (mr > 0 ? mr : 1);
}

static float* up(const std::vector<float>& h) {
    float* d = nullptr;
    cudaMalloc(&d, h.size() * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    return d;
}
static std::vector<float> down(const float* d, size_t n) {
    std::vector<float> h(n);
    cudaMemcpy(h.data(), d, n * 4, cudaMemcpyDeviceToHost);
    return h;
}

int main() {
    const uint32_t F = 16, H = 2, W = 4, C = 64, taps = 3, G = 8;
    const size_t n = size_t(F) * H * W * C;
    std::vector<float> x(n), sa(C), sc(C), cw(taps * C * C), cb(C), ga(C), be(C), wq(C * C),
        wk(C * C), wv(C * C), wo(C * C), want(n);
    orc_fill_seeded(x.data(), n, 5, 0, 1.0f);
    orc_build_block(C, taps, 1, 0, sa.data(), sc.data(), cw.data(), cb.data(), ga.data(),
                    be.data(), wq.data(), wk.data(), wv.data(), wo.data());
    float *dx = up(x), *dy = nullptr;
    cudaMalloc(&dy, n * 4);
    b::DeviceTensor tx{dx, F, H, W, C, VINF_F32}, ty{dy, F, H, W, C, VINF_F32};
    int fails = 0;

    // temporal_conv (ops.cpp:106-108)
    b::ConvKernel k(taps, C, up(cw), up(cb));
    b::temporal_conv(tx, k, ty);
    orc_conv_over_extended(x.data(), F, H, W, C, 0, F, taps, cw.data(), cb.data(), want.data());
    double e = normwise(down(dy, n), want);
    std::printf("temporal_conv normwise %.3e\n", e);
    fails += !(e <= 1e-4);

    // group_norm (ops.cpp:169-173)
    b::GroupNormParams gp{G, up(ga), up(be), 1e-5f};
    b::group_norm(tx, gp, ty);
    orc_group_norm(x.data(), n, C, G, ga.data(), be.data(), 1e-5f, want.data());
    e = normwise(down(dy, n), want);
    std::printf("group_norm normwise %.3e\n", e);
    fails += !(e <= 1e-5);

    // dual_scope_reference (ops.cpp:291-338)
    const float scale = 1.0f / std::sqrt(float(C));
    b::AttentionParams ap(C, scale, up(wq), up(wk), up(wv), up(wo));
    b::DualScopeConfig cfg{8, 4, 10.0f, 800.0};
    b::dual_scope_reference(tx, 900.0, ap, cfg, ty);
    orc_dual_scope(x.data(), F, H, W, C, 900.0, wq.data(), wk.data(), wv.data(), wo.data(), scale,
                   1, 8, 4, 10.0f, 800.0, want.data(), nullptr);
    e = normwise(down(dy, n), want);
    std::printf("dual_scope normwise %.3e\n", e);
    fails += !(e <= 1e-4);

    // token sets and the error taxonomy
    const auto g = b::build_global_index_set(24, 16);
    fails += !(g.size() == 16 && g[2] == 3 && g[15] == 22);
    try {
        b::GroupNormParams bad{3, gp.gamma, gp.beta, 1e-5f};
        b::group_norm(tx, bad, ty);
        fails += 1;
    } catch (const b::ConfigError&) {
    }
    try {
        b::make_plan(2300, 8);
        fails += 1;
    } catch (const b::ConfigError&) {
    }
    try {
        b::ClipPlan plan = b::make_plan(16, 2);
        b::DeviceTensor half{dx, 8, H, W, C, VINF_F32};
        b::conv_parallel(plan, 1, half, b::TemporalContext{}, k, ty);  // worker 1 needs c_pre
        fails += 1;
    } catch (const b::ProtocolError&) {
    }
    std::printf("%s (%d failures)\n", fails ? "FAIL" : "PASS", fails);
    return fails ? 1 : 0;
}
