// Run-level C ABI (include/vinf_run.h): the reference's outer API (include/vinf.h:27-75)
// over the clip engine. Configuration handling restates config.cpp (keys, defaults,
// canonical text, FNV-1a digest, violations); execution restates runner.cpp's dispatch
// and pipeline.cpp's worker loop with one device engine per worker; dumps follow
// tensor_io.cpp and metrics records metrics.cpp:40-85.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/vinf_run.h"
#include "host.hpp"

namespace vinf {
int guarded_call(const std::function<void()>& f);
extern thread_local std::string g_last_error;

namespace run {

[[noreturn]] void io_error(const std::string& m) { throw Error(VINF_ERR_IO, m); }

// ---- configuration (config.hpp:17-40 fields and defaults) ---------------------------

struct RunConfig {
    uint32_t frames = 16, height = 4, width = 4, channels = 8, workers = 1;
    uint32_t blocks = 1, taps = 3, groups = 2, n_local = 16, n_global = 16;
    double bias = 10.0, t_star = 800.0;
    uint32_t steps = 30;
    uint64_t seed = 0, weight_seed = 1;
    std::string transport = "inproc", listen = "127.0.0.1:45600";
    bool validating = false, sequential = false;
    std::string ablate = "none";
    std::string dtype = "f32";  // extension: device arithmetic (f32 | bf16)
};

std::string trim(const std::string& s) {
    const char* ws = " \t\r\n";
    const size_t b = s.find_first_not_of(ws);
    if (b == std::string::npos) return "";
    return s.substr(b, s.find_last_not_of(ws) - b + 1);
}

uint64_t to_u64(const std::string& k, const std::string& v) {
    size_t used = 0;
    uint64_t x = 0;
    bool ok = !v.empty() && v[0] != '-';
    if (ok) {
        try {
            x = std::stoull(v, &used);
        } catch (...) {
            ok = false;
        }
    }
    if (!ok || used != v.size()) config_error("value for '" + k + "' is not an integer: " + v);
    return x;
}
uint32_t to_u32(const std::string& k, const std::string& v) {
    const uint64_t x = to_u64(k, v);
    if (x > 0xffffffffull) config_error("value for '" + k + "' out of range: " + v);
    return uint32_t(x);
}
double to_f64(const std::string& k, const std::string& v) {
    size_t used = 0;
    double x = 0;
    bool ok = !v.empty();
    if (ok) {
        try {
            x = std::stod(v, &used);
        } catch (...) {
            ok = false;
        }
    }
    if (!ok || used != v.size()) config_error("value for '" + k + "' is not a number: " + v);
    return x;
}
bool to_bool(const std::string& k, const std::string& v) {
    if (v == "true" || v == "1") return true;
    if (v == "false" || v == "0") return false;
    config_error("value for '" + k + "' must be true or false: " + v);
}

void set_key(RunConfig& c, const std::string& key_raw, const std::string& value_raw) {
    const std::string k = trim(key_raw), v = trim(value_raw);
    struct U32 { const char* name; uint32_t RunConfig::*field; };
    static const U32 u32s[] = {{"frames", &RunConfig::frames},   {"height", &RunConfig::height},
                               {"width", &RunConfig::width},     {"channels", &RunConfig::channels},
                               {"workers", &RunConfig::workers}, {"blocks", &RunConfig::blocks},
                               {"taps", &RunConfig::taps},       {"groups", &RunConfig::groups},
                               {"n_local", &RunConfig::n_local}, {"n_global", &RunConfig::n_global},
                               {"steps", &RunConfig::steps}};
    for (const U32& f : u32s)
        if (k == f.name) {
            c.*(f.field) = to_u32(k, v);
            return;
        }
    if (k == "bias") c.bias = to_f64(k, v);
    else if (k == "t_star") c.t_star = to_f64(k, v);
    else if (k == "seed") c.seed = to_u64(k, v);
    else if (k == "weight_seed") c.weight_seed = to_u64(k, v);
    else if (k == "transport") c.transport = v;
    else if (k == "listen") c.listen = v;
    else if (k == "validating") c.validating = to_bool(k, v);
    else if (k == "sequential") c.sequential = to_bool(k, v);
    else if (k == "ablate") c.ablate = v;
    else if (k == "dtype") c.dtype = v;
    else config_error("unknown config key: " + k);
}

RunConfig parse_text(const std::string& text) {
    RunConfig c;
    std::istringstream in(text);
    std::string line;
    for (size_t no = 1; std::getline(in, line); ++no) {
        const size_t hash = line.find('#');
        if (hash != std::string::npos) line.resize(hash);
        line = trim(line);
        if (line.empty()) continue;
        const size_t eq = line.find('=');
        if (eq == std::string::npos)
            config_error("config line " + std::to_string(no) + " has no '=': " + line);
        set_key(c, line.substr(0, eq), line.substr(eq + 1));
    }
    return c;
}

std::string f64_text(double v) {
    char b[40];
    snprintf(b, sizeof(b), "%.17g", v);
    return b;
}

// Every key, sorted, one per line (config.cpp:143-171); the dtype extension only when it
// differs from its default, so reference configurations digest identically.
std::string canonical(const RunConfig& c) {
    std::vector<std::pair<std::string, std::string>> kv = {
        {"ablate", c.ablate},
        {"bias", f64_text(c.bias)},
        {"blocks", std::to_string(c.blocks)},
        {"channels", std::to_string(c.channels)},
        {"frames", std::to_string(c.frames)},
        {"groups", std::to_string(c.groups)},
        {"height", std::to_string(c.height)},
        {"listen", c.listen},
        {"n_global", std::to_string(c.n_global)},
        {"n_local", std::to_string(c.n_local)},
        {"seed", std::to_string(c.seed)},
        {"sequential", c.sequential ? "true" : "false"},
        {"steps", std::to_string(c.steps)},
        {"t_star", f64_text(c.t_star)},
        {"taps", std::to_string(c.taps)},
        {"transport", c.transport},
        {"validating", c.validating ? "true" : "false"},
        {"weight_seed", std::to_string(c.weight_seed)},
        {"width", std::to_string(c.width)},
        {"workers", std::to_string(c.workers)}};
    if (c.dtype != "f32") kv.push_back({"dtype", c.dtype});
    std::sort(kv.begin(), kv.end());
    std::string out;
    for (const auto& [k, v] : kv) out += k + "=" + v + "\n";
    return out;
}

uint64_t fnv1a64(const std::string& s) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (unsigned char ch : s) h = (h ^ ch) * 0x100000001b3ull;
    return h;
}

std::vector<std::string> violations(const RunConfig& c) {
    std::vector<std::string> v;
    auto need = [&](bool ok, const std::string& msg) {
        if (!ok) v.push_back(msg);
    };
    auto s = [](uint64_t x) { return std::to_string(x); };
    need(c.frames >= 1, "frames must be >= 1");
    need(c.height >= 1, "height must be >= 1");
    need(c.width >= 1, "width must be >= 1");
    need(c.channels >= 1, "channels must be >= 1");
    need(c.workers >= 1, "workers must be >= 1");
    need(c.blocks >= 1, "blocks must be >= 1");
    need(c.steps >= 1, "steps must be >= 1");
    need(c.taps % 2 == 1, "taps must be odd and >= 1 (got " + s(c.taps) + ")");
    need(c.groups != 0 && (c.channels == 0 || c.channels % c.groups == 0),
         "groups must divide channels (groups=" + s(c.groups) + " channels=" + s(c.channels) + ")");
    need(c.n_local >= 2 && c.n_local % 2 == 0,
         "n_local must be even and >= 2 (got " + s(c.n_local) + ")");
    need(c.n_global <= c.frames, "n_global must not exceed frames (n_global=" + s(c.n_global) +
                                     " frames=" + s(c.frames) + ")");
    need(c.bias >= 0, "bias must be >= 0");
    if (c.workers != 0 && c.frames % c.workers != 0) {
        v.push_back("workers must divide frames evenly (frames=" + s(c.frames) +
                    " workers=" + s(c.workers) + ")");
    } else if (c.workers != 0 && c.frames != 0) {
        const uint32_t fc = c.frames / c.workers;
        need(c.taps / 2 <= fc, "conv halo exceeds clip ((taps-1)/2=" + s(c.taps / 2) +
                                   " > frames/workers=" + s(fc) + ")");
        need(c.n_local / 2 <= fc, "attention halo exceeds clip (n_local/2=" + s(c.n_local / 2) +
                                      " > frames/workers=" + s(fc) + ")");
    }
    need(c.transport == "inproc" || c.transport == "tcp",
         "transport must be inproc or tcp (got '" + c.transport + "')");
    if (c.transport == "tcp") {
        const size_t colon = c.listen.rfind(':');
        bool ok = colon != std::string::npos && colon > 0 && colon + 1 < c.listen.size();
        for (size_t i = ok ? colon + 1 : c.listen.size(); i < c.listen.size(); ++i)
            ok = ok && c.listen[i] >= '0' && c.listen[i] <= '9';
        need(ok, "listen must be host:port (got '" + c.listen + "')");
    }
    need(c.ablate == "none" || c.ablate == "conv" || c.ablate == "groupnorm" ||
             c.ablate == "attention",
         "ablate must be none, conv, groupnorm, or attention (got '" + c.ablate + "')");
    need(c.dtype == "f32" || c.dtype == "bf16", "dtype must be f32 or bf16 (got '" + c.dtype + "')");
    // Limits of the device backend that the reference (CPU) does not have; listed after the
    // reference's own checks so a config it rejects reports the same messages first
    // (INTEGRATION.md §4): 16-byte TMA rows and the attention core's K/V tile.
    need(c.channels == 0 || c.channels % 8 == 0,
         "device backend: channels must be a multiple of 8 (got " + s(c.channels) + ")");
    need(uint64_t(c.n_local) + 1 + c.n_global <= uint64_t(kMaxTokens),
         "device backend: n_local + 1 + n_global must be <= " + s(kMaxTokens) + " (got " +
             s(uint64_t(c.n_local) + 1 + c.n_global) + ")");
    return v;
}

void validate(const RunConfig& c) {
    const auto v = violations(c);
    if (v.empty()) return;
    std::string msg = "invalid config:";
    for (const auto& m : v) msg += "\n  - " + m;
    config_error(msg);
}

int ablate_kind(const std::string& a) {
    if (a == "conv") return VINF_ABLATE_CONV;
    if (a == "groupnorm") return VINF_ABLATE_GROUPNORM;
    if (a == "attention") return VINF_ABLATE_ATTENTION;
    return VINF_ABLATE_NONE;
}
const char* kind_name(int k) {
    return k == VINF_ABLATE_CONV ? "conv" : k == VINF_ABLATE_GROUPNORM ? "groupnorm" : "attention";
}

// ---- tensor dumps (tensor_io.cpp) ----------------------------------------------------

struct Dump {
    uint32_t f = 0, h = 0, w = 0, c = 0;
    std::vector<float> data;
};

void put32(std::string& s, uint32_t v) {
    for (int i = 0; i < 4; ++i) s.push_back(char((v >> (8 * i)) & 0xff));
}
uint32_t get32(const unsigned char* p) {
    return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
}

void write_dump(const std::string& path, const Dump& d) {
    std::string hdr = "VINF";
    put32(hdr, 1);
    for (uint32_t x : {d.f, d.h, d.w, d.c}) put32(hdr, x);
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) io_error("cannot open for writing: " + path);
    out.write(hdr.data(), std::streamsize(hdr.size()));
    out.write(reinterpret_cast<const char*>(d.data.data()), std::streamsize(d.data.size() * 4));
    if (!out) io_error("write failed: " + path);
}

Dump read_dump(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) io_error("cannot open for reading: " + path);
    unsigned char h[24];
    in.read(reinterpret_cast<char*>(h), 24);
    if (in.gcount() != 24) io_error("truncated dump header: " + path);
    if (std::memcmp(h, "VINF", 4) != 0) io_error("bad magic in dump: " + path);
    if (get32(h + 4) != 1) io_error("unsupported dump version " + std::to_string(get32(h + 4)) + ": " + path);
    Dump d;
    d.f = get32(h + 8), d.h = get32(h + 12), d.w = get32(h + 16), d.c = get32(h + 20);
    if (!d.f || !d.h || !d.w || !d.c) shape_error("invalid shape in dump: " + path);
    d.data.resize(uint64_t(d.f) * d.h * d.w * d.c);
    in.read(reinterpret_cast<char*>(d.data.data()), std::streamsize(d.data.size() * 4));
    if (uint64_t(in.gcount()) != d.data.size() * 4) io_error("truncated dump payload: " + path);
    char extra;
    if (in.read(&extra, 1)) io_error("trailing bytes after dump payload: " + path);
    return d;
}

// ---- execution ---------------------------------------------------------------------

struct KindStats {
    uint64_t calls = 0, msgs = 0, bytes = 0, contributed = 0;
    double t1 = 0, t2 = 0, t3 = 0;
};
struct WorkerStats {
    KindStats kind[3];  // conv, groupnorm, attention
    uint64_t score_entries = 0, queries = 0, max_tokens = 0, bias_global = 0, bias_local = 0;
    int64_t peak_live = 0;
    double wall = 0;
};
struct RunResult {
    Dump x0;
    std::vector<WorkerStats> workers;
    double wall = 0;
};

void ck(cudaError_t e, const char* what) { cuda_check(int(e), what); }

// One engine per worker on the current device; exchanges are copies between workspaces.
struct Job {
    struct Copy { uint8_t* dst; const uint8_t* src; uint64_t bytes; };
    uint32_t n = 1;
    cudaStream_t s = nullptr;
    std::vector<vinf_layout*> layouts;
    std::vector<vinf_engine*> engines;
    std::vector<uint8_t*> ws;
    std::vector<std::vector<Copy>> copies[2];      // [stage][worker] receive copies
    std::vector<uint64_t> sent_msgs[2], sent_bytes[2];
    std::vector<uint64_t> sums_off;  // per worker: edge workers' layouts differ
    uint64_t sums_bytes = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;

    ~Job() {
        if (s) cudaStreamSynchronize(s);
        for (auto* e : engines) vinf_engine_destroy(e);
        for (auto* p : ws) cudaFree(p);
        for (auto* l : layouts) vinf_layout_destroy(l);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (s) cudaStreamDestroy(s);
    }

    void check(int rc) {
        if (rc != VINF_OK) throw Error(rc, g_last_error);
    }

    void plan_exchanges() {
        for (int st = 0; st < 2; ++st) {
            std::vector<std::vector<vinf_xfer>> xs(n);
            for (uint32_t w = 0; w < n; ++w) {
                uint32_t cnt = 0;
                check(vinf_layout_exchange(layouts[w], st, nullptr, 0, &cnt));
                xs[w].resize(cnt);
                if (cnt) check(vinf_layout_exchange(layouts[w], st, xs[w].data(), cnt, &cnt));
            }
            copies[st].assign(n, {});
            sent_msgs[st].assign(n, 0);
            sent_bytes[st].assign(n, 0);
            for (uint32_t w = 0; w < n; ++w)
                for (const vinf_xfer& x : xs[w]) {
                    if (x.send) {
                        sent_msgs[st][w] += 1;
                        sent_bytes[st][w] += x.bytes;
                        continue;
                    }
                    const vinf_xfer* src = nullptr;
                    for (const vinf_xfer& y : xs[x.peer])
                        if (y.send && y.peer == w && y.tag == x.tag) src = &y;
                    if (!src || src->bytes != x.bytes)
                        protocol_error("unmatched transfer into worker " + std::to_string(w));
                    copies[st][w].push_back({ws[w] + x.offset, ws[x.peer] + src->offset, x.bytes});
                }
        }
    }

    double exchange(int st) {  // device milliseconds of the exchange
        ck(cudaEventRecord(ev0, s), "event");
        for (uint32_t w = 0; w < n; ++w)
            for (const Copy& c : copies[st][w])
                ck(cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyDeviceToDevice, s), "exchange");
        ck(cudaEventRecord(ev1, s), "event");
        ck(cudaEventSynchronize(ev1), "exchange sync");
        float ms = 0;
        cudaEventElapsedTime(&ms, ev0, ev1);
        return ms;
    }

    double allreduce_sums(uint32_t groups) {  // sum in worker order, like LocalGroup
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<double> total(2 * groups, 0.0), part(2 * groups);
        ck(cudaStreamSynchronize(s), "sums sync");
        // all copies on the job's (non-blocking) stream: a legacy-stream cudaMemcpy from
        // pageable memory may return before its DMA lands
        for (uint32_t w = 0; w < n; ++w) {
            ck(cudaMemcpyAsync(part.data(), ws[w] + sums_off[w], sums_bytes, cudaMemcpyDeviceToHost, s), "sums");
            ck(cudaStreamSynchronize(s), "sums sync");
            for (size_t i = 0; i < total.size(); ++i) total[i] = w == 0 ? part[i] : total[i] + part[i];
        }
        for (uint32_t w = 0; w < n; ++w)
            ck(cudaMemcpyAsync(ws[w] + sums_off[w], total.data(), sums_bytes, cudaMemcpyHostToDevice, s), "sums");
        ck(cudaStreamSynchronize(s), "sums sync");
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
};

RunResult execute(const RunConfig& c) {
    validate(c);
    if (c.transport == "tcp")
        config_error("transport=tcp is not provided by the device backend: its workers are clip "
                     "engines on this GPU (transport=inproc); multi-GPU runs use torch.distributed "
                     "over NCCL (paper_2406_16260_b200.engine.DistGroup)");
    const uint32_t n = c.sequential ? 1 : c.workers;
    const uint32_t f_clip = c.frames / n;
    const vinf_dtype dt = c.dtype == "bf16" ? VINF_BF16 : VINF_F32;
    const int ablate = c.sequential ? VINF_ABLATE_NONE : ablate_kind(c.ablate);
    const uint64_t E = uint64_t(c.height) * c.width * c.channels;

    Job job;
    job.n = n;
    ck(cudaStreamCreateWithFlags(&job.s, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreate(&job.ev0), "event");
    ck(cudaEventCreate(&job.ev1), "event");
    uint64_t ws_bytes = 0;
    for (uint32_t w = 0; w < n; ++w) {
        vinf_engine_desc d{};
        d.frames = c.frames;
        d.workers = n;
        d.worker = w;
        d.height = c.height;
        d.width = c.width;
        d.channels = c.channels;
        d.taps = c.taps;
        d.groups = c.groups;
        d.heads = 1;
        d.n_local = c.n_local;
        d.n_global = c.n_global;
        d.bias = float(c.bias);
        d.t_star = c.t_star;
        d.epsilon = 1e-5f;
        d.scale = 0.f;
        d.blocks = c.blocks;
        d.dtype = dt;
        vinf_layout* l = nullptr;
        job.check(vinf_layout_create(&d, &l));
        job.layouts.push_back(l);
        job.check(vinf_layout_workspace_bytes(l, &ws_bytes));
        uint8_t* p = nullptr;
        ck(cudaMalloc(&p, ws_bytes), "workspace");
        job.ws.push_back(p);
        vinf_engine* e = nullptr;
        job.check(vinf_engine_create(l, p, job.s, &e));
        job.engines.push_back(e);
        job.check(vinf_engine_init_weights(e, c.weight_seed, job.s));
        job.check(vinf_engine_set_ablation(e, ablate));
    }
    job.sums_off.assign(n, 0);
    for (uint32_t w = 0; w < n; ++w) {
        uint64_t fb = 0;
        job.check(vinf_layout_region(job.layouts[w], VINF_BUF_GN_SUMS, &job.sums_off[w], &job.sums_bytes, &fb));
    }
    job.plan_exchanges();

    // attention counters per call (ops.cpp:327-333): tokens per query frame
    std::vector<uint64_t> tok_w(n, 0), tok_max(n, 0);
    for (uint32_t w = 0; w < n; ++w)
        for (uint32_t a = w * f_clip; a < (w + 1) * f_clip; ++a) {
            const uint64_t t = build_local_window(a, c.frames, c.n_local).size() + c.n_global;
            tok_w[w] += t;
            tok_max[w] = std::max(tok_max[w], t);
        }

    RunResult res;
    res.workers.assign(n, {});
    const uint32_t hw = c.height * c.width;
    const auto t0 = std::chrono::steady_clock::now();
    for (uint32_t w = 0; w < n; ++w) {
        void *x = nullptr, *y = nullptr;
        job.check(vinf_engine_io(job.engines[w], &x, &y));
        job.check(vinf_fill_seeded(x, dt, uint64_t(f_clip) * E, c.seed, uint64_t(w) * f_clip * E, 1.0f, job.s));
    }
    for (uint32_t j = c.steps; j >= 1; --j) {  // timestep_grid (pipeline.cpp:75-81)
        const double t = 1000.0 * j / c.steps;
        for (uint32_t b = 0; b < c.blocks; ++b) {
            for (auto* e : job.engines) job.check(vinf_engine_stage(e, b, VINF_STAGE_STUB, t, job.s));
            const uint64_t call = c.sequential ? 0 : 1;  // the sequential oracle never syncs
            for (uint32_t w = 0; w < n; ++w) res.workers[w].kind[0].calls += call;
            if (n > 1 && ablate != VINF_ABLATE_CONV) {
                const double ms = job.exchange(VINF_XCHG_CONV);
                for (uint32_t w = 0; w < n; ++w) {
                    KindStats& k = res.workers[w].kind[0];
                    k.msgs += job.sent_msgs[0][w];
                    k.bytes += job.sent_bytes[0][w];
                    k.contributed += job.sent_bytes[0][w];
                    k.t1 += ms * 1e-3;
                }
            }
            for (auto* e : job.engines) job.check(vinf_engine_stage(e, b, VINF_STAGE_CONV, t, job.s));
            for (uint32_t w = 0; w < n; ++w) res.workers[w].kind[1].calls += call;
            if (n > 1 && ablate != VINF_ABLATE_GROUPNORM) {
                const double sec = job.allreduce_sums(c.groups);
                for (uint32_t w = 0; w < n; ++w) {
                    KindStats& k = res.workers[w].kind[1];
                    k.msgs += n - 1;
                    k.bytes += uint64_t(2) * c.groups * 8 * (n - 1);
                    k.contributed += uint64_t(2) * c.groups * 8;
                    k.t1 += sec;
                }
            }
            for (auto* e : job.engines) job.check(vinf_engine_stage(e, b, VINF_STAGE_GN_APPLY, t, job.s));
            for (uint32_t w = 0; w < n; ++w) res.workers[w].kind[2].calls += call;
            if (n > 1 && ablate != VINF_ABLATE_ATTENTION) {
                const double ms = job.exchange(VINF_XCHG_ATTN);
                for (uint32_t w = 0; w < n; ++w) {
                    KindStats& k = res.workers[w].kind[2];
                    k.msgs += job.sent_msgs[1][w];
                    k.bytes += job.sent_bytes[1][w];
                    k.contributed += job.sent_bytes[1][w];
                    k.t1 += ms * 1e-3;
                }
            }
            for (auto* e : job.engines) job.check(vinf_engine_stage(e, b, VINF_STAGE_ATTENTION, t, job.s));
            for (uint32_t w = 0; w < n; ++w) {
                WorkerStats& ws = res.workers[w];
                ws.queries += uint64_t(f_clip) * hw;
                ws.score_entries += tok_w[w] * hw;
                ws.max_tokens = tok_max[w];
            }
        }
        for (auto* e : job.engines) job.check(vinf_engine_euler(e, 1.0 / c.steps, job.s));
        for (uint32_t w = 0; w < n; ++w) (t > c.t_star ? res.workers[w].bias_global : res.workers[w].bias_local) += 1;
    }
    ck(cudaStreamSynchronize(job.s), "run sync");
    res.wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

    res.x0 = Dump{c.frames, c.height, c.width, c.channels, std::vector<float>(uint64_t(c.frames) * E)};
    std::vector<uint16_t> tmp(dt == VINF_BF16 ? uint64_t(f_clip) * E : 0);
    for (uint32_t w = 0; w < n; ++w) {
        void *x = nullptr, *y = nullptr;
        job.check(vinf_engine_io(job.engines[w], &x, &y));
        float* dst = res.x0.data.data() + uint64_t(w) * f_clip * E;
        if (dt == VINF_F32) {
            ck(cudaMemcpy(dst, x, uint64_t(f_clip) * E * 4, cudaMemcpyDeviceToHost), "x0");
        } else {
            ck(cudaMemcpy(tmp.data(), x, tmp.size() * 2, cudaMemcpyDeviceToHost), "x0");
            for (size_t i = 0; i < tmp.size(); ++i) {
                const uint32_t bits = uint32_t(tmp[i]) << 16;
                std::memcpy(dst + i, &bits, 4);
            }
        }
        res.workers[w].peak_live = int64_t(ws_bytes / 4);
        res.workers[w].wall = res.wall;
    }
    return res;
}

std::string records(const RunConfig& c, const RunResult& r, const std::string& label) {
    std::string out;
    char b[512];
    snprintf(b, sizeof(b), "run digest=0x%016llx workers=%u transport=%s label=%s steps=%u wall_s=%.6f\n",
             (unsigned long long)fnv1a64(canonical(c)), c.sequential ? 1u : c.workers,
             c.sequential ? "sequential" : c.transport.c_str(), label.c_str(), c.steps, r.wall);
    out += b;
    for (uint32_t i = 0; i < r.workers.size(); ++i) {
        const WorkerStats& w = r.workers[i];
        for (int k = 0; k < 3; ++k) {
            const KindStats& s = w.kind[k];
            snprintf(b, sizeof(b),
                     "sync worker=%u kind=%s calls=%llu msgs=%llu bytes_sent=%llu "
                     "bytes_contributed=%llu t1_s=%.6f t2_s=%.6f t3_s=%.6f\n",
                     i, kind_name(k + 1), (unsigned long long)s.calls, (unsigned long long)s.msgs,
                     (unsigned long long)s.bytes, (unsigned long long)s.contributed, s.t1, s.t2, s.t3);
            out += b;
        }
        snprintf(b, sizeof(b),
                 "worker id=%u peak_live=%lld score_entries=%llu queries=%llu max_tokens=%llu "
                 "bias_global=%llu bias_local=%llu wall_s=%.6f\n",
                 i, (long long)w.peak_live, (unsigned long long)w.score_entries,
                 (unsigned long long)w.queries, (unsigned long long)w.max_tokens,
                 (unsigned long long)w.bias_global, (unsigned long long)w.bias_local, w.wall);
        out += b;
    }
    return out;
}

void write_outputs(const RunConfig& c, const RunResult& r, const char* out_path,
                   const char* metrics_path, const std::string& label) {
    if (out_path && *out_path) write_dump(out_path, r.x0);
    if (metrics_path && *metrics_path) {
        std::ofstream m(metrics_path, std::ios::app);
        if (!m) io_error(std::string("cannot open metrics file: ") + metrics_path);
        m << records(c, r, label);
        if (!m) io_error(std::string("metrics write failed: ") + metrics_path);
    }
}

double max_abs_diff(const std::vector<float>& a, const std::vector<float>& b) {
    double m = 0;
    for (size_t i = 0; i < a.size() && i < b.size(); ++i)
        m = std::max(m, std::fabs(double(a[i]) - double(b[i])));
    return m;
}

std::string bench(const RunConfig& base, const std::vector<uint32_t>& sweep, const char* metrics) {
    struct Row {
        std::string label;
        uint32_t workers;
        double wall, speedup, maxd;
        uint64_t bytes[3];
        bool diverged;
    };
    std::vector<Row> rows;
    RunConfig seq = base;
    seq.sequential = true;
    seq.workers = 1;
    seq.ablate = "none";
    const RunResult br = execute(seq);
    write_outputs(seq, br, nullptr, metrics, "bench sequential");
    auto row = [&](const std::string& label, const RunConfig& c, const RunResult& r) {
        Row x{label, c.sequential ? 1u : c.workers, r.wall, r.wall > 0 ? br.wall / r.wall : 0.0,
              max_abs_diff(r.x0.data, br.x0.data), {0, 0, 0}, false};
        for (const WorkerStats& w : r.workers)
            for (int k = 0; k < 3; ++k) x.bytes[k] += w.kind[k].bytes;
        x.diverged = x.maxd > double(c.steps) * 1e-5;  // runner.cpp:256-258
        rows.push_back(x);
    };
    row("sequential", seq, br);
    for (uint32_t n : sweep) {
        RunConfig c = base;
        c.sequential = false;
        c.workers = n;
        c.ablate = "none";
        const std::string label = "n=" + std::to_string(n);
        const RunResult r = execute(c);
        write_outputs(c, r, nullptr, metrics, "bench " + label);
        row(label, c, r);
        if (n <= 1) continue;
        for (int k = VINF_ABLATE_CONV; k <= VINF_ABLATE_ATTENTION; ++k) {
            RunConfig a = c;
            a.ablate = kind_name(k);
            const std::string al = label + " -" + kind_name(k) + "-sync";
            const RunResult ar = execute(a);
            write_outputs(a, ar, nullptr, metrics, "bench " + al);
            row(al, a, ar);
        }
    }
    std::string out;
    char b[256];
    snprintf(b, sizeof(b), "%-28s %7s %9s %8s %12s %12s %12s %10s %8s\n", "label", "workers", "wall_s",
             "speedup", "conv_B", "gnorm_B", "attn_B", "max_diff", "diverged");
    out += b;
    for (const Row& r : rows) {
        snprintf(b, sizeof(b), "%-28s %7u %9.3f %8.2f %12llu %12llu %12llu %10.3g %8s\n", r.label.c_str(),
                 r.workers, r.wall, r.speedup, (unsigned long long)r.bytes[0],
                 (unsigned long long)r.bytes[1], (unsigned long long)r.bytes[2], r.maxd,
                 r.diverged ? "yes" : "no");
        out += b;
    }
    return out;
}

// ---- schedule simulation (schedule.cpp) ------------------------------------------

struct Op {
    bool send;
    uint32_t peer;
};

// Ring edge i -> i+1 is coloured by parity; with an odd worker count the wrap edge
// would clash with edge 0 at worker 0 and takes a third colour. A worker issues the
// lower-coloured of its two ring operations first.
std::vector<std::vector<Op>> shipped_schedule(uint32_t n) {
    std::vector<std::vector<Op>> prog(n);
    if (n == 1) return prog;
    auto colour = [n](uint32_t edge) { return (n % 2 == 1 && edge == n - 1) ? 2u : edge % 2; };
    for (uint32_t i = 0; i < n; ++i) {
        const uint32_t to = (i + 1) % n, from = (i + n - 1) % n;
        const bool send_first = colour(i) < colour(from);
        for (uint32_t r = 1; r < n; ++r) {
            const Op s{true, to}, v{false, from};
            prog[i].push_back(send_first ? s : v);
            prog[i].push_back(send_first ? v : s);
        }
        for (uint32_t parity = 0; parity < 2; ++parity) {  // pair stages T2, T3
            if (i % 2 == parity && i + 1 < n) {
                prog[i].push_back({true, i + 1});
                prog[i].push_back({false, i + 1});
            } else if (i >= 1 && (i - 1) % 2 == parity) {
                prog[i].push_back({false, i - 1});
                prog[i].push_back({true, i - 1});
            }
        }
    }
    return prog;
}

// The published pseudocode's pair order: receive first on both sides.
std::vector<std::vector<Op>> literal_schedule(uint32_t n) {
    std::vector<std::vector<Op>> prog(n);
    for (uint32_t i = 0; i < n; ++i) {
        const int64_t first = i % 2 == 1 ? int64_t(i) + 1 : int64_t(i) - 1;
        const int64_t second = i % 2 == 1 ? int64_t(i) - 1 : int64_t(i) + 1;
        for (int64_t p : {first, second})
            if (p >= 0 && p < int64_t(n)) {
                prog[i].push_back({false, uint32_t(p)});
                prog[i].push_back({true, uint32_t(p)});
            }
    }
    return prog;
}

struct Verdict {
    bool completed = false;
    uint32_t rounds = 0;
    uint64_t transfers = 0;
    std::vector<uint32_t> cycle;
};

// Strict rendezvous, one transfer per worker per round: fire a maximal set of disjoint
// matched (send i->j, recv j<-i) pairs, scanning senders in index order.
Verdict simulate(const std::vector<std::vector<Op>>& prog) {
    const uint32_t n = uint32_t(prog.size());
    std::vector<size_t> pc(n, 0);
    auto done = [&](uint32_t i) { return pc[i] >= prog[i].size(); };
    Verdict v;
    for (;;) {
        bool all = true;
        for (uint32_t i = 0; i < n; ++i) all = all && done(i);
        if (all) {
            v.completed = true;
            return v;
        }
        std::vector<uint8_t> busy(n, 0);
        uint64_t fired = 0;
        for (uint32_t i = 0; i < n; ++i) {
            if (done(i) || !prog[i][pc[i]].send) continue;
            const uint32_t j = prog[i][pc[i]].peer;
            if (j >= n || j == i || done(j) || busy[i] || busy[j]) continue;
            const Op& o = prog[j][pc[j]];
            if (o.send || o.peer != i) continue;
            busy[i] = busy[j] = 1;
            ++fired;
        }
        if (fired == 0) {
            // deadlock: follow wait-for edges (every blocked op waits on its peer)
            std::vector<int> seen(n, -1);
            for (uint32_t s0 = 0; s0 < n; ++s0) {
                if (done(s0) || seen[s0] >= 0) continue;
                std::vector<uint32_t> path;
                uint32_t cur = s0;
                while (cur < n && !done(cur) && seen[cur] < 0) {
                    seen[cur] = int(path.size());
                    path.push_back(cur);
                    cur = prog[cur][pc[cur]].peer;
                }
                if (cur < n && !done(cur) && seen[cur] >= 0 && size_t(seen[cur]) < path.size() &&
                    path[size_t(seen[cur])] == cur) {
                    v.cycle.assign(path.begin() + seen[cur], path.end());
                    return v;
                }
            }
            return v;
        }
        for (uint32_t i = 0; i < n; ++i)
            if (busy[i]) ++pc[i];
        v.rounds += 1;
        v.transfers += fired;
    }
}

void fill_text(const std::string& text, char* buf, size_t cap, size_t* needed) {
    if (needed) *needed = text.size();
    if (buf && cap > 0) {
        const size_t k = std::min(text.size(), cap - 1);
        std::memcpy(buf, text.data(), k);
        buf[k] = '\0';
    }
}

}  // namespace run
}  // namespace vinf

struct vinf_config {
    vinf::run::RunConfig cfg;
};

using namespace vinf;

extern "C" {

int vinf_config_create(vinf_config** out) {
    return guarded_call([&] {
        if (!out) shape_error("vinf_config_create: out is NULL");
        *out = new vinf_config();
    });
}

void vinf_config_destroy(vinf_config* cfg) { delete cfg; }

int vinf_config_load_file(vinf_config* cfg, const char* path) {
    return guarded_call([&] {
        if (!cfg || !path) shape_error("vinf_config_load_file: NULL argument");
        std::ifstream in(path);
        if (!in) run::io_error(std::string("cannot open config file: ") + path);
        std::ostringstream text;
        text << in.rdbuf();
        cfg->cfg = run::parse_text(text.str());
    });
}

int vinf_config_set(vinf_config* cfg, const char* key, const char* value) {
    return guarded_call([&] {
        if (!cfg || !key || !value) shape_error("vinf_config_set: NULL argument");
        run::set_key(cfg->cfg, key, value);
    });
}

int vinf_config_validate(const vinf_config* cfg) {
    return guarded_call([&] {
        if (!cfg) shape_error("vinf_config_validate: cfg is NULL");
        run::validate(cfg->cfg);
    });
}

int vinf_config_digest(const vinf_config* cfg, uint64_t* digest_out) {
    return guarded_call([&] {
        if (!cfg || !digest_out) shape_error("vinf_config_digest: NULL argument");
        *digest_out = run::fnv1a64(run::canonical(cfg->cfg));
    });
}

int vinf_config_canonical(const vinf_config* cfg, char* buf, size_t cap, size_t* needed) {
    return guarded_call([&] {
        if (!cfg) shape_error("vinf_config_canonical: cfg is NULL");
        run::fill_text(run::canonical(cfg->cfg), buf, cap, needed);
    });
}

int vinf_run(const vinf_config* cfg, const char* out_path, const char* metrics_path,
             double* wall_seconds_out) {
    return guarded_call([&] {
        if (!cfg) shape_error("vinf_run: cfg is NULL");
        const run::RunResult r = run::execute(cfg->cfg);
        run::write_outputs(cfg->cfg, r, out_path, metrics_path, "run");
        if (wall_seconds_out) *wall_seconds_out = r.wall;
    });
}

int vinf_verify(const char* dump_a, const char* dump_b, double tolerance, double* max_diff_out,
                uint64_t* mismatch_count_out) {
    return guarded_call([&] {
        if (!dump_a || !dump_b) shape_error("vinf_verify: NULL path");
        const run::Dump a = run::read_dump(dump_a), b = run::read_dump(dump_b);
        if (a.f != b.f || a.h != b.h || a.w != b.w || a.c != b.c)
            shape_error(std::string("shape mismatch between '") + dump_a + "' and '" + dump_b + "'");
        double md = 0;
        uint64_t bad = 0;
        for (size_t i = 0; i < a.data.size(); ++i) {
            const double d = std::fabs(double(a.data[i]) - double(b.data[i]));
            md = std::max(md, d);
            bad += d > tolerance;
        }
        if (max_diff_out) *max_diff_out = md;
        if (mismatch_count_out) *mismatch_count_out = bad;
        if (bad) throw Error(VINF_ERR, "dumps differ beyond tolerance");
    });
}

int vinf_bench(const vinf_config* cfg, const uint32_t* sweep, size_t sweep_len,
               const char* metrics_path, char* table_buf, size_t table_cap,
               size_t* table_needed) {
    return guarded_call([&] {
        if (!cfg || (sweep_len > 0 && !sweep)) shape_error("vinf_bench: NULL argument");
        const std::vector<uint32_t> counts(sweep, sweep + sweep_len);
        run::fill_text(run::bench(cfg->cfg, counts, metrics_path), table_buf, table_cap, table_needed);
    });
}

int vinf_validate_schedule(uint32_t workers, int literal_order, int* completed_out,
                           uint32_t* rounds_out, uint64_t* transfers_out, char* cycle_buf,
                           size_t cycle_cap) {
    return guarded_call([&] {
        if (workers == 0) shape_error("vinf_validate_schedule: workers must be >= 1");
        const run::Verdict v = run::simulate(literal_order ? run::literal_schedule(workers)
                                                           : run::shipped_schedule(workers));
        if (completed_out) *completed_out = v.completed ? 1 : 0;
        if (rounds_out) *rounds_out = v.rounds;
        if (transfers_out) *transfers_out = v.transfers;
        std::string cyc;
        for (size_t i = 0; i < v.cycle.size(); ++i) cyc += (i ? " -> " : "") + std::to_string(v.cycle[i]);
        if (!v.cycle.empty()) cyc += " -> " + std::to_string(v.cycle.front());
        run::fill_text(cyc, cycle_buf, cycle_cap, nullptr);
    });
}

}  // extern "C"
