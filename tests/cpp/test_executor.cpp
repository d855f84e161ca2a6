// The clip-parallel worker loop as a reference maintainer writes it against the C ABI
// (INTEGRATION.md §2): N worker threads, each with its own layout, workspace, engine and
// stream, running worker_denoise (pipeline.cpp:174-191) with the 3-step context sync through
// the library's executor (vinf_engine_denoise_dist over in-process communicators, the shape of
// the reference's run_inproc_workers, transport_inproc.cpp:148-189). The denoised clip must
// match a single worker's run within the reference's cross-worker invariance bar
// (acceptance c4, acceptance.cpp:228-260: 3e-4 after 30 steps). Built and run by
// tests/test_cpp_mirror.py.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <thread>
#include <vector>

#include "vinf_temporal.h"

#define CHECK(x)                                                                                  \
    do {                                                                                          \
        const int rc_ = (x);                                                                      \
        if (rc_ != VINF_OK) {                                                                     \
            std::printf("FAIL %s -> %d: %s\n", #x, rc_, vinf_last_error());                     \
            return 1;                                                                             \
        }                                                                                         \
    } while (0)

struct Worker {
    vinf_layout* L = nullptr;
    vinf_engine* E = nullptr;
    void* ws = nullptr;
    cudaStream_t s = nullptr;
    uint32_t start = 0, frames = 0;
};

static vinf_engine_desc desc(uint32_t F, uint32_t N, uint32_t w, vinf_dtype dt) {
    vinf_engine_desc d{};
    d.frames = F;
    d.workers = N;
    d.worker = w;
    d.height = 2;
    d.width = 8;
    d.channels = 64;
    d.taps = 3;
    d.groups = 8;
    d.heads = 1;
    d.n_local = 8;
    d.n_global = 8;
    d.bias = 10.0f;
    d.t_star = 800.0;
    d.epsilon = 1e-5f;
    d.scale = 0.f;
    d.blocks = 2;
    d.dtype = dt;
    d.uneven = 0;
    return d;
}

static int make(Worker& wk, const vinf_engine_desc& d) {
    CHECK(vinf_layout_create(&d, &wk.L));
    uint64_t bytes = 0;
    CHECK(vinf_layout_workspace_bytes(wk.L, &bytes));
    CHECK(vinf_layout_clip(wk.L, &wk.start, &wk.frames));
    if (cudaStreamCreateWithFlags(&wk.s, cudaStreamNonBlocking) != cudaSuccess) return 1;
    if (cudaMalloc(&wk.ws, bytes) != cudaSuccess) return 1;
    CHECK(vinf_engine_create(wk.L, wk.ws, wk.s, &wk.E));
    CHECK(vinf_engine_init_weights(wk.E, 1, wk.s));
    void* x = nullptr;
    CHECK(vinf_engine_io(wk.E, &x, nullptr));
    const uint64_t e = uint64_t(d.height) * d.width * d.channels;
    // this worker's frames of tensor_from_seed({F,H,W,C}, 0) (runner.cpp:59-60)
    CHECK(vinf_fill_seeded(x, d.dtype, uint64_t(wk.frames) * e, 0, uint64_t(wk.start) * e, 1.0f, wk.s));
    return 0;
}

static std::vector<float> result(const Worker& wk, uint64_t n) {
    void* x = nullptr;
    vinf_engine_io(wk.E, &x, nullptr);
    std::vector<float> h(n);
    cudaStreamSynchronize(wk.s);
    cudaMemcpy(h.data(), x, n * 4, cudaMemcpyDeviceToHost);
    return h;
}

int main() {
    const uint32_t F = 48, N = 3, steps = 30;
    const uint64_t e = 2 * 8 * 64;
    // single worker: the whole video, no sync (vinf_engine_denoise)
    Worker one;
    if (make(one, desc(F, 1, 0, VINF_F32))) return 1;
    CHECK(vinf_engine_denoise(one.E, steps, one.s));
    const std::vector<float> want = result(one, uint64_t(F) * e);

    // N workers, one host thread each, the executor over in-process communicators
    std::vector<Worker> ws(N);
    for (uint32_t w = 0; w < N; ++w)
        if (make(ws[w], desc(F, N, w, VINF_F32))) return 1;
    std::vector<vinf_comm*> comms(N);
    CHECK(vinf_comm_create_local(N, comms.data()));
    std::vector<int> rcs(N, 0);
    std::vector<std::thread> th;
    for (uint32_t w = 0; w < N; ++w)
        th.emplace_back([&, w] {
            rcs[w] = vinf_engine_denoise_dist(ws[w].E, steps, comms[w], 1, ws[w].s);
            if (rcs[w] != VINF_OK) {
                std::printf("worker %u: %s\n", w, vinf_last_error());
                vinf_comm_abort(comms[w]);
            }
        });
    for (auto& t : th) t.join();
    for (uint32_t w = 0; w < N; ++w)
        if (rcs[w] != VINF_OK) return 1;
    double md = 0, mr = 0;
    uint64_t sent = 0;
    for (uint32_t w = 0; w < N; ++w) {
        const std::vector<float> got = result(ws[w], uint64_t(ws[w].frames) * e);
        for (uint64_t i = 0; i < got.size(); ++i) {
            const double ref = want[uint64_t(ws[w].start) * e + i];
            md = std::fmax(md, std::fabs(double(got[i]) - ref));
            mr = std::fmax(mr, std::fabs(ref));
        }
        uint64_t b = 0;
        CHECK(vinf_comm_info(comms[w], nullptr, nullptr, &b, nullptr));
        sent += b;
    }
    const double err = md / (mr > 0 ? mr : 1);
    std::printf("executor: %u workers x %u frames, %u steps, 2 blocks: x0 normwise vs 1 worker %.3e, %llu bytes sent\n",
                N, F / N, steps, err, static_cast<unsigned long long>(sent));
    for (auto* c : comms) vinf_comm_destroy(c);
    if (!(err <= 3e-4) || sent == 0) {
        std::printf("FAIL\n");
        return 1;
    }
    std::printf("PASS\n");
    return 0;
}
