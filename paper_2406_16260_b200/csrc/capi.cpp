// C ABI (include/vinf_temporal.h): guarded wrappers mapping the internal error taxonomy
// to status codes with a thread-local last-error message, as the reference's capi.cpp
// (guarded, capi.cpp:22-48) does for its run-level API.
#include <cuda_runtime.h>

#include <cstring>
#include <functional>
#include <string>

#include "host.hpp"
#include "layout.hpp"
#include "ops.hpp"

namespace vinf {

thread_local std::string g_last_error;

int guarded_call(const std::function<void()>& f) {
    try {
        f();
        return VINF_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "out of host memory";
        return VINF_ERR;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return VINF_ERR;
    }
}

uint64_t mix_seed(uint64_t seed, uint64_t salt);

namespace {
void copy_out(const std::vector<uint32_t>& v, uint32_t* out, uint32_t cap, uint32_t* count) {
    if (count) *count = uint32_t(v.size());
    if (v.size() > cap) range_error("output capacity too small");
    if (!v.empty()) {
        if (!out) shape_error("null output buffer");
        std::memcpy(out, v.data(), v.size() * sizeof(uint32_t));
    }
}
cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
}  // namespace

}  // namespace vinf

using namespace vinf;

extern "C" {

const char* vinf_version(void) { return "vinf-b200 0.1.0 (sm_100a)"; }
const char* vinf_last_error(void) { return g_last_error.c_str(); }

int vinf_device_ok(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return 0;
    }
    int dev = 0, major = 0, minor = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    return (major == 10 && minor == 0) ? 1 : 0;
}

int vinf_build_local_window(uint32_t a, uint32_t frames, uint32_t n_local, uint32_t* out,
                            uint32_t cap, uint32_t* count) {
    return guarded_call([&] { copy_out(build_local_window(a, frames, n_local), out, cap, count); });
}

int vinf_build_global_index_set(uint32_t frames, uint32_t n_global, uint32_t* out, uint32_t cap,
                                uint32_t* count) {
    return guarded_call(
        [&] { copy_out(build_global_index_set(frames, n_global), out, cap, count); });
}

int vinf_make_plan(uint32_t frames, uint32_t workers, uint32_t* f_clip) {
    return guarded_call([&] {
        const uint32_t f = make_plan(frames, workers);
        if (f_clip) *f_clip = f;
    });
}

int vinf_global_members_in_range(uint32_t frames, uint32_t n_global, uint32_t start,
                                 uint32_t len, uint32_t* out, uint32_t cap, uint32_t* count) {
    return guarded_call([&] {
        copy_out(global_members_in_range(frames, n_global, start, len), out, cap, count);
    });
}

int vinf_predict_sync_traffic(uint32_t frames, uint32_t workers, uint32_t halo,
                              uint32_t global_frames, uint32_t worker, uint64_t frame_bytes,
                              uint64_t* out3) {
    return guarded_call([&] {
        if (!out3) shape_error("null output");
        if (worker >= workers) range_error("worker index out of range");
        predict_sync_traffic(frames, workers, halo, global_frames, worker, frame_bytes, out3);
    });
}

int vinf_predict_groupnorm_traffic(uint32_t frames, uint32_t workers, uint32_t groups,
                                   uint32_t worker, uint64_t* out3) {
    return guarded_call([&] {
        if (!out3) shape_error("null output");
        if (worker >= workers) range_error("worker index out of range");
        predict_groupnorm_traffic(frames, workers, groups, out3);
    });
}

int vinf_fill_seeded(void* dst, vinf_dtype dtype, uint64_t n, uint64_t seed, uint64_t first_elem,
                     float scale, void* stream) {
    return guarded_call([&] {
        if (!dst && n) shape_error("null destination");
        cuda_check(launch_fill_seeded(dst, dtype == VINF_BF16, n, seed, first_elem, scale, S(stream)),
                   "fill_seeded");
    });
}

uint64_t vinf_mix_seed(uint64_t seed, uint64_t salt) { return mix_seed(seed, salt); }

// ---- parameter handles ----

int vinf_conv_kernel_create(uint32_t taps, uint32_t channels, const float* weights,
                            const float* bias, vinf_conv_kernel** out) {
    return guarded_call([&] {
        if (!out) shape_error("null output");
        if (taps == 0 || taps % 2 == 0)
            config_error("conv taps must be odd and >= 1, got " + std::to_string(taps));
        if (channels == 0 || !weights || !bias) shape_error("conv kernel sized for wrong channel count");
        auto* k = new vinf_conv_kernel();
        k->taps = taps;
        k->C = channels;
        k->w.alloc(taps * channels, channels);
        k->w.from_f32(weights, nullptr);
        cuda_check(cudaMalloc(&k->bias, sizeof(float) * channels), "cudaMalloc(bias)");
        cuda_check(cudaMemcpy(k->bias, bias, sizeof(float) * channels, cudaMemcpyDeviceToDevice),
                   "bias copy");
        cuda_check(cudaDeviceSynchronize(), "conv kernel create");
        *out = k;
    });
}

void vinf_conv_kernel_destroy(vinf_conv_kernel* k) {
    if (!k) return;
    k->w.release();
    if (k->bias) cudaFree(k->bias);
    delete k;
}

int vinf_attention_params_create(uint32_t dim, uint32_t heads, float scale, const float* wq,
                                 const float* wk, const float* wv, const float* wo,
                                 vinf_attention_params** out) {
    return guarded_call([&] {
        if (!out) shape_error("null output");
        if (dim == 0 || !wq || !wk || !wv || !wo) shape_error("attention projections must be C x C");
        if (heads == 0 || dim % heads != 0) config_error("heads must divide dim");
        if (!(scale > 0.0f)) config_error("attention scale must be > 0");
        auto* p = new vinf_attention_params();
        p->C = dim;
        p->heads = heads;
        p->scale = scale;
        const size_t m = size_t(dim) * dim;
        float* tmp = nullptr;
        cuda_check(cudaMalloc(&tmp, 3 * m * sizeof(float)), "cudaMalloc(tmp)");
        cuda_check(cudaMemcpy(tmp, wq, m * 4, cudaMemcpyDeviceToDevice), "wq");
        cuda_check(cudaMemcpy(tmp + m, wk, m * 4, cudaMemcpyDeviceToDevice), "wk");
        cuda_check(cudaMemcpy(tmp + 2 * m, wv, m * 4, cudaMemcpyDeviceToDevice), "wv");
        p->wqkv.alloc(3 * dim, dim);
        p->wqkv.from_f32(tmp, nullptr);
        p->wo.alloc(dim, dim);
        p->wo.from_f32(wo, nullptr);
        cuda_check(cudaDeviceSynchronize(), "attention params create");
        cudaFree(tmp);
        *out = p;
    });
}

void vinf_attention_params_destroy(vinf_attention_params* p) {
    if (!p) return;
    p->wqkv.release();
    p->wo.release();
    delete p;
}

// ---- operators ----

int vinf_spatial_affine_tanh(const vinf_tensor* v, const float* a, const float* c,
                             vinf_tensor* out, void* stream) {
    return guarded_call([&] {
        check_tensor(v, "stub input");
        check_tensor(out, "stub output");
        if (!a || !c) shape_error("stub coeffs must have C entries");
        if (numel(v) != numel(out) || v->c != out->c) shape_error("stub output shape mismatch");
        cuda_check(launch_stub(v->data, v->dtype == VINF_BF16, numel(v), v->c, a, c, out->data,
                               out->dtype == VINF_BF16, nullptr, nullptr, S(stream)),
                   "stub");
    });
}

int vinf_conv_over_extended(const vinf_tensor* ext, uint32_t out_start, uint32_t out_len,
                            const vinf_conv_kernel* k, vinf_tensor* out, void* stream) {
    return guarded_call([&] { conv_over_extended(ext, out_start, out_len, k, out, S(stream)); });
}

int vinf_temporal_conv(const vinf_tensor* v, const vinf_conv_kernel* k, vinf_tensor* out,
                       void* stream) {
    return guarded_call([&] {
        if (!v) shape_error("null tensor");
        conv_over_extended(v, 0, v->f, k, out, S(stream));
    });
}

int vinf_group_means(const vinf_tensor* v, uint32_t groups, double* means, void* stream) {
    return guarded_call([&] { group_stat(v, groups, nullptr, means, S(stream)); });
}

int vinf_group_sqdev(const vinf_tensor* v, uint32_t groups, const double* means, double* vars,
                     void* stream) {
    return guarded_call([&] {
        if (!means) shape_error("means must have one entry per group");
        group_stat(v, groups, means, vars, S(stream));
    });
}

int vinf_group_partial_sums(const vinf_tensor* v, uint32_t groups, const double* center,
                            double* sums, void* stream) {
    return guarded_call([&] { group_sums(v, groups, center, sums, S(stream)); });
}

int vinf_normalize_with_stats(const vinf_tensor* v, const vinf_group_norm_params* p,
                              const double* means, const double* vars, vinf_tensor* out,
                              void* stream) {
    return guarded_call([&] {
        if (!means || !vars) shape_error("stats must have one entry per group");
        normalize_with_stats(v, p, means, vars, out, S(stream));
    });
}

int vinf_group_norm(const vinf_tensor* v, const vinf_group_norm_params* p, vinf_tensor* out,
                    void* stream) {
    return guarded_call([&] { group_norm(v, p, out, S(stream)); });
}

int vinf_dual_scope_attention(const vinf_tensor* v, double t, const vinf_attention_params* p,
                              const vinf_dual_scope_config* cfg, vinf_tensor* out, void* stream) {
    return guarded_call([&] { dual_scope(v, t, p, cfg, out, S(stream)); });
}

int vinf_attention_full(const vinf_tensor* v, const vinf_attention_params* p, vinf_tensor* out,
                        void* stream) {
    return guarded_call([&] { attention_full(v, p, out, S(stream)); });
}

int vinf_conv_parallel(uint32_t frames, uint32_t workers, uint32_t worker, const vinf_tensor* v,
                       const vinf_tensor* ctx_pre, const vinf_tensor* ctx_post,
                       const vinf_conv_kernel* k, vinf_tensor* out, void* stream) {
    return guarded_call([&] {
        conv_parallel(frames, workers, worker, v, ctx_pre, ctx_post, k, out, S(stream));
    });
}

int vinf_attention_parallel(uint32_t frames, uint32_t workers, uint32_t worker,
                            const vinf_tensor* v, const vinf_tensor* ctx_pre,
                            const vinf_tensor* ctx_post, const vinf_tensor* ctx_global, double t,
                            const vinf_attention_params* p, const vinf_dual_scope_config* cfg,
                            vinf_tensor* out, void* stream) {
    return guarded_call([&] {
        attention_parallel(frames, workers, worker, v, ctx_pre, ctx_post, ctx_global, t, p, cfg,
                           out, S(stream));
    });
}

// ---- diagnostics ----

int vinf_gemm_bench(uint32_t M, uint32_t N, uint32_t K, uint32_t nseg, int flags, int residual,
                    int iters, float* avg_ms) {
    return guarded_call([&] {
        if (!M || !N || !K || !nseg || iters <= 0 || !avg_ms) shape_error("bad gemm bench args");
        cudaStream_t s = nullptr;
        const uint64_t arows = uint64_t(M) + uint64_t(nseg) * 64;
        TmpBuf a(arows * K * 2, s), o(uint64_t(M) * N * 2, s), r(residual ? uint64_t(M) * N * 2 : 0, s);
        DevMat B;
        B.alloc(nseg * N, K);
        cuda_check(launch_fill_seeded(a.p, true, arows * K, 1, 0, 1.0f, s), "fill");
        cuda_check(launch_fill_seeded(B.hi, true, uint64_t(nseg) * N * K, 2, 0, 0.03f, s), "fill");
        if (residual) cuda_check(launch_fill_seeded(r.p, true, uint64_t(M) * N, 3, 0, 1.0f, s), "fill");
        Operand A;
        A.hi = static_cast<const __nv_bfloat16*>(a.p);
        A.rows = arows;
        A.cols = K;
        A.ld = K;
        std::vector<int64_t> ar, br;
        for (uint32_t j = 0; j < nseg; ++j) {
            ar.push_back(int64_t(j) * 64);
            br.push_back(int64_t(j) * N);
        }
        Epilogue ep;
        ep.out = o.p;
        ep.out_ld = N;
        ep.out_bf16 = true;
        if (residual) {
            ep.res = r.p;
            ep.res_ld = N;
            ep.res_bf16 = true;
        }
        g_gemm_debug_flags = flags;
        for (int i = 0; i < 2; ++i) gemm(A, ar, B, br, M, N, ep, false, s);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, s);
        for (int i = 0; i < iters; ++i) gemm(A, ar, B, br, M, N, ep, false, s);
        cudaEventRecord(e1, s);
        cuda_check(cudaEventSynchronize(e1), "gemm bench");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        *avg_ms = ms / iters;
        if (flags & 2) {  // determinism check: compare 5 further runs against this output
            const size_t nb = uint64_t(M) * N * 2;
            std::vector<uint8_t> ref(nb), cur(nb);
            cuda_check(cudaMemcpy(ref.data(), o.p, nb, cudaMemcpyDeviceToHost), "copy");
            uint64_t bad = 0;
            for (int rep = 0; rep < 5; ++rep) {
                gemm(A, ar, B, br, M, N, ep, false, s);
                cuda_check(cudaMemcpy(cur.data(), o.p, nb, cudaMemcpyDeviceToHost), "copy");
                for (size_t i = 0; i < nb; i += 2)
                    bad += (ref[i] != cur[i] || ref[i + 1] != cur[i + 1]) ? 1 : 0;
            }
            *avg_ms = -float(bad);  // report mismatching elements instead of time
        }
        g_gemm_debug_flags = 0;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        B.release();
    });
}

// ---- layout ----

int vinf_layout_create(const vinf_engine_desc* d, vinf_layout** out) {
    return guarded_call([&] {
        if (!d || !out) shape_error("null argument");
        *out = new vinf_layout(*d);
    });
}

void vinf_layout_destroy(vinf_layout* l) { delete l; }

int vinf_layout_workspace_bytes(const vinf_layout* l, uint64_t* bytes) {
    return guarded_call([&] {
        if (!l || !bytes) shape_error("null argument");
        *bytes = l->L.total;
    });
}

int vinf_layout_region(const vinf_layout* l, int which, uint64_t* offset, uint64_t* bytes,
                       uint64_t* frame_bytes) {
    return guarded_call([&] {
        if (!l) shape_error("null layout");
        const Layout& L = l->L;
        uint64_t off = 0, n = 0, fb = L.E * L.es;
        switch (which) {
            case VINF_BUF_X: off = L.off_x; n = uint64_t(L.f_clip) * fb; break;
            case VINF_BUF_Y: off = L.off_y; n = uint64_t(L.f_clip) * fb; break;
            case VINF_BUF_CONV_IN: fb = L.E * 2; off = L.off_u0; n = uint64_t(L.cf) * fb; break;
            case VINF_BUF_ATTN_IN: fb = L.E * 2; off = L.off_u2; n = uint64_t(L.af) * fb; break;
            case VINF_BUF_GN_SUMS: fb = 0; off = L.off_sums; n = 2 * 8 * uint64_t(L.d.groups); break;
            case VINF_BUF_QKV: fb = L.E * 3 * L.es; off = L.off_qkv; n = uint64_t(L.af) * fb; break;
            case VINF_BUF_CTX: fb = L.E * 2; off = L.off_ctx; n = uint64_t(L.f_clip) * fb; break;
            default: range_error("unknown region");
        }
        if (offset) *offset = off;
        if (bytes) *bytes = n;
        if (frame_bytes) *frame_bytes = fb;
    });
}

int vinf_layout_clip(const vinf_layout* l, uint32_t* start, uint32_t* frames) {
    return guarded_call([&] {
        if (!l) shape_error("null layout");
        if (start) *start = l->L.start;
        if (frames) *frames = l->L.f_clip;
    });
}

int vinf_layout_exchange(const vinf_layout* l, int stage, vinf_xfer* out, uint32_t cap,
                         uint32_t* count) {
    return guarded_call([&] {
        if (!l) shape_error("null layout");
        const auto& xs = stage == VINF_XCHG_CONV ? l->L.xconv : l->L.xattn;
        if (stage != VINF_XCHG_CONV && stage != VINF_XCHG_ATTN) range_error("unknown stage");
        if (count) *count = uint32_t(xs.size());
        if (!out && cap == 0) return;  // size query
        if (xs.size() > cap) range_error("output capacity too small");
        if (!xs.empty()) std::memcpy(out, xs.data(), xs.size() * sizeof(vinf_xfer));
    });
}

int vinf_layout_reference_traffic(const vinf_layout* l, uint64_t* conv3, uint64_t* gn3,
                                  uint64_t* attn3) {
    return guarded_call([&] {
        if (!l) shape_error("null layout");
        const Layout& L = l->L;
        const uint64_t fb = L.E * 4;  // the reference moves fp32 frames
        if (conv3) predict_sync_traffic(L.d.frames, L.d.workers, L.hc, 0, L.d.worker, fb, conv3);
        if (gn3) predict_groupnorm_traffic(L.d.frames, L.d.workers, L.d.groups, gn3);
        if (attn3)
            predict_sync_traffic(L.d.frames, L.d.workers, L.ha, L.d.n_global, L.d.worker, fb, attn3);
    });
}

}  // extern "C"
