// Diagnostics (not on the product path): micro-benchmarks of the attention core on a
// single-worker engine layout's token table, and a streaming-read bandwidth probe.
#include <cuda_runtime.h>

#include <cstdlib>
#include <functional>
#include <string>
#include <vector>

#include "host.hpp"
#include "layout.hpp"
#include "ops.hpp"

namespace vinf {
int guarded_call(const std::function<void()>& f);
int read_bw_bench(uint64_t bytes, int iters, float* ms);
int bulk_bw_bench(uint64_t bytes, uint32_t chunk, uint32_t stages, uint32_t ctas, int iters, float* ms);
}  // namespace vinf

using namespace vinf;

extern "C" {

int vinf_read_bw_bench(uint64_t bytes, int iters, float* ms) {
    return guarded_call([&] {
        if (!ms || iters <= 0 || bytes < 16) shape_error("bad arguments");
        cuda_check(read_bw_bench(bytes, iters, ms), "read bandwidth probe");
    });
}

int vinf_bulk_bw_bench(uint64_t bytes, uint32_t chunk, uint32_t stages, uint32_t ctas, int iters, float* ms) {
    return guarded_call([&] {
        if (!ms || iters <= 0 || chunk % 16 || !stages) shape_error("bad arguments");
        cuda_check(bulk_bw_bench(bytes, chunk, stages, ctas, iters, ms), "bulk bandwidth probe");
    });
}

// Selects the attention core implementation for later launches (0 = by configuration,
// 1 = TMA ring, 2 = cp.async ring); returns the previous setting.
int vinf_debug_attention_impl(int impl) {
    const int old = g_attn_impl;
    if (impl >= 0 && impl <= 2) g_attn_impl = impl;
    return old;
}

// The attention core alone over the Q/K/V buffer of a single-worker engine layout
// (t > t_star token table), average ms over iters launches; pos_major must be 0 (the
// frame-major [frames][HW][3C] buffer; the other layouts were measured and removed).
int vinf_attention_bench(uint32_t frames, uint32_t height, uint32_t width, uint32_t channels, uint32_t heads,
                         uint32_t n_local, uint32_t n_global, int f32, int pos_major, int iters, float* ms) {
    return guarded_call([&] {
        if (!ms || iters <= 0) shape_error("bad arguments");
        if (pos_major) shape_error("pos_major: only the frame-major layout is built (DESIGN.md section 3)");
        vinf_engine_desc d{};
        d.frames = frames;
        d.workers = 1;
        d.height = height;
        d.width = width;
        d.channels = channels;
        d.taps = 3;
        d.groups = 8;
        d.heads = heads;
        d.n_local = n_local;
        d.n_global = n_global;
        d.bias = 10.f;
        d.t_star = 800.0;
        d.epsilon = 1e-5f;
        d.blocks = 1;
        d.dtype = f32 ? VINF_F32 : VINF_BF16;
        Layout L(d);
        DevTokens tok;
        cudaStream_t s = nullptr;
        cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
        tok.upload(L.tok[1], s);
        {  // the buffers are freed (stream-ordered) before the stream is destroyed
        const uint64_t plane = uint64_t(L.af) * L.hw * 3 * channels;
        const uint64_t ctxn = uint64_t(L.f_clip) * L.hw * channels;
        TmpBuf qkv(plane * 2 * (f32 ? 2 : 1), s), ctx(ctxn * 2 * (f32 ? 2 : 1), s);
        cuda_check(cudaMemsetAsync(qkv.p, 0x3c, plane * 2 * (f32 ? 2 : 1), s), "fill");
        // VINF_DIAG_FUSE=1 (one head): the fused output (block output = ctx' + res * s + t)
        const bool fuse = getenv("VINF_DIAG_FUSE") && heads == 1;
        TmpBuf res(fuse ? ctxn * (f32 ? 4 : 2) : 16, s), aff(fuse ? 2ull * channels * 4 : 16, s),
            yb(fuse ? ctxn * (f32 ? 4 : 2) : 16, s);
        FuseO fo;
        if (fuse) {
            cuda_check(cudaMemsetAsync(res.p, 0x3c, ctxn * (f32 ? 4 : 2), s), "fill");
            cuda_check(cudaMemsetAsync(aff.p, 0, 2ull * channels * 4, s), "fill");
            fo.res = res.p;
            fo.res_bf16 = !f32;
            if (!f32) {
                fo.s = static_cast<const float*>(aff.p);
                fo.t = static_cast<const float*>(aff.p) + channels;
            }
            fo.y = yb.p;
            fo.y_bf16 = !f32;
        }
        auto* q = static_cast<__nv_bfloat16*>(qkv.p);
        auto* c = static_cast<__nv_bfloat16*>(ctx.p);
        auto launch = [&] {
            cuda_check(launch_attention_core(q, f32 ? q + plane : nullptr, L.af, L.hw, channels, heads, L.f_clip,
                                             L.ha, tok.tt, L.scale, d.bias, c, f32 ? c + ctxn : nullptr, s, &fo),
                       "attention core");
        };
        launch();
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, s);
        for (int i = 0; i < iters; ++i) launch();
        cudaEventRecord(b, s);
        cuda_check(cudaEventSynchronize(b), "attention bench");
        cudaEventElapsedTime(ms, a, b);
        *ms /= float(iters);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        }
        cuda_check(cudaStreamSynchronize(s), "sync");
        tok.release();
        cudaStreamDestroy(s);
    });
}

}  // extern "C"
