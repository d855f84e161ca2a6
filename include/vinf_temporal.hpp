// vinf_temporal.hpp — header-only C++ mirror of the reference temporal-module API over
// the C ABI (vinf_temporal.h). Same names, argument meaning and error behaviour as
// /root/reference/proj/src/core/ops.hpp:49-124 and clip_parallel.hpp:14-84, but on DEVICE
// tensors: a reference caller swaps `vinf::temporal_conv(t, k)` for
// `vinf::b200::temporal_conv(t, k)` with t a DeviceTensor. Errors are thrown as the
// reference's exception types (error.hpp:10-34), mapped from the C status codes.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "vinf_temporal.h"

namespace vinf {
namespace b200 {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ConfigError : Error {  // error.hpp:12
    using Error::Error;
};
struct ShapeError : Error {  // error.hpp:16 (also RangeError)
    using Error::Error;
};
struct TransportError : Error {  // error.hpp:29
    using Error::Error;
};
struct ProtocolError : TransportError {  // error.hpp:33
    using TransportError::TransportError;
};

inline void check(int rc) {
    if (rc == VINF_OK) return;
    const std::string msg = vinf_last_error();
    switch (rc) {
        case VINF_ERR_CONFIG: throw ConfigError(msg);
        case VINF_ERR_INVALID: throw ShapeError(msg);
        case VINF_ERR_TRANSPORT: throw ProtocolError(msg);
        default: throw Error(msg);
    }
}

// Dims + device pointer (tensor.hpp:15-24 layout: [F,H,W,C], channels innermost).
struct DeviceTensor {
    void* data = nullptr;
    uint32_t f = 0, h = 0, w = 0, c = 0;
    vinf_dtype dtype = VINF_F32;
    bool empty() const { return f == 0 || data == nullptr; }
    size_t frame_elems() const { return size_t(h) * w * c; }
    size_t total() const { return size_t(f) * frame_elems(); }
    vinf_tensor c_view() const { return vinf_tensor{data, f, h, w, c, dtype}; }
};

class ConvKernel {  // ops.hpp:14-21 (weights/bias: device fp32)
   public:
    ConvKernel(uint32_t taps, uint32_t channels, const float* weights_dev, const float* bias_dev) {
        vinf_conv_kernel* k = nullptr;
        check(vinf_conv_kernel_create(taps, channels, weights_dev, bias_dev, &k));
        h_.reset(k);
        taps_ = taps;
    }
    uint32_t halo() const { return (taps_ - 1) / 2; }
    const vinf_conv_kernel* get() const { return h_.get(); }

   private:
    struct Del {
        void operator()(vinf_conv_kernel* k) const { vinf_conv_kernel_destroy(k); }
    };
    std::unique_ptr<vinf_conv_kernel, Del> h_;
    uint32_t taps_ = 1;
};

class AttentionParams {  // ops.hpp:32-36 (+ heads extension)
   public:
    AttentionParams(uint32_t dim, float scale, const float* wq, const float* wk, const float* wv,
                    const float* wo, uint32_t heads = 1) {
        vinf_attention_params* p = nullptr;
        check(vinf_attention_params_create(dim, heads, scale, wq, wk, wv, wo, &p));
        h_.reset(p);
    }
    const vinf_attention_params* get() const { return h_.get(); }

   private:
    struct Del {
        void operator()(vinf_attention_params* p) const { vinf_attention_params_destroy(p); }
    };
    std::unique_ptr<vinf_attention_params, Del> h_;
};

using GroupNormParams = vinf_group_norm_params;  // ops.hpp:23-30 (gamma/beta device)
using DualScopeConfig = vinf_dual_scope_config;  // ops.hpp:38-43

// ---- token sets / plan (ops.cpp:177-198, clip_parallel.cpp:54-91) ----
inline std::vector<uint32_t> build_local_window(uint32_t a, uint32_t frames, uint32_t n_local) {
    std::vector<uint32_t> out(n_local + 2);
    uint32_t n = 0;
    check(vinf_build_local_window(a, frames, n_local, out.data(), uint32_t(out.size()), &n));
    out.resize(n);
    return out;
}
inline std::vector<uint32_t> build_global_index_set(uint32_t frames, uint32_t n_global) {
    std::vector<uint32_t> out(n_global ? n_global : 1);
    uint32_t n = 0;
    check(vinf_build_global_index_set(frames, n_global, out.data(), uint32_t(out.size()), &n));
    out.resize(n);
    return out;
}
struct ClipPlan {  // clip_parallel.hpp:14-19
    uint32_t n = 1, f = 0, f_clip = 0;
};
inline ClipPlan make_plan(uint32_t frames, uint32_t workers) {
    ClipPlan p;
    check(vinf_make_plan(frames, workers, &p.f_clip));
    p.n = workers;
    p.f = frames;
    return p;
}

// ---- operators (ops.cpp). `out` is caller-allocated, shaped like the reference result. ----
inline void temporal_conv(const DeviceTensor& v, const ConvKernel& k, DeviceTensor& out,
                          void* stream = nullptr) {
    const vinf_tensor a = v.c_view();
    vinf_tensor o = out.c_view();
    check(vinf_temporal_conv(&a, k.get(), &o, stream));
}
inline void conv_over_extended(const DeviceTensor& ext, uint32_t out_start, uint32_t out_len,
                               const ConvKernel& k, DeviceTensor& out, void* stream = nullptr) {
    const vinf_tensor a = ext.c_view();
    vinf_tensor o = out.c_view();
    check(vinf_conv_over_extended(&a, out_start, out_len, k.get(), &o, stream));
}
inline void group_norm(const DeviceTensor& v, const GroupNormParams& p, DeviceTensor& out,
                       void* stream = nullptr) {
    const vinf_tensor a = v.c_view();
    vinf_tensor o = out.c_view();
    check(vinf_group_norm(&a, &p, &o, stream));
}
inline void dual_scope_reference(const DeviceTensor& v, double t, const AttentionParams& p,
                                 const DualScopeConfig& cfg, DeviceTensor& out,
                                 void* stream = nullptr) {
    const vinf_tensor a = v.c_view();
    vinf_tensor o = out.c_view();
    check(vinf_dual_scope_attention(&a, t, p.get(), &cfg, &o, stream));
}
inline void attention_full(const DeviceTensor& v, const AttentionParams& p, DeviceTensor& out,
                           void* stream = nullptr) {
    const vinf_tensor a = v.c_view();
    vinf_tensor o = out.c_view();
    check(vinf_attention_full(&a, p.get(), &o, stream));
}

// ---- distributed forms (clip_parallel.cpp:194-341) ----
struct TemporalContext {  // clip_parallel.hpp:40-44 (empty tensors at the video edge)
    DeviceTensor c_pre, c_post, c_global;
};
inline void conv_parallel(const ClipPlan& plan, uint32_t worker, const DeviceTensor& v,
                          const TemporalContext& ctx, const ConvKernel& k, DeviceTensor& out,
                          void* stream = nullptr) {
    const vinf_tensor a = v.c_view(), pre = ctx.c_pre.c_view(), post = ctx.c_post.c_view();
    vinf_tensor o = out.c_view();
    check(vinf_conv_parallel(plan.f, plan.n, worker, &a, ctx.c_pre.empty() ? nullptr : &pre,
                             ctx.c_post.empty() ? nullptr : &post, k.get(), &o, stream));
}
inline void attention_parallel(const ClipPlan& plan, uint32_t worker, const DeviceTensor& v,
                               const TemporalContext& ctx, double t, const AttentionParams& p,
                               const DualScopeConfig& cfg, DeviceTensor& out,
                               void* stream = nullptr) {
    const vinf_tensor a = v.c_view(), pre = ctx.c_pre.c_view(), post = ctx.c_post.c_view(),
                      g = ctx.c_global.c_view();
    vinf_tensor o = out.c_view();
    check(vinf_attention_parallel(plan.f, plan.n, worker, &a, ctx.c_pre.empty() ? nullptr : &pre,
                                  ctx.c_post.empty() ? nullptr : &post,
                                  ctx.c_global.empty() ? nullptr : &g, t, p.get(), &cfg, &o,
                                  stream));
}

}  // namespace b200
}  // namespace vinf
