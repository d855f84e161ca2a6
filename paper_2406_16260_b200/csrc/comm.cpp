// Communicators (comm.hpp): NCCL over NVLink/NVSwitch, in-process workers, and
// caller-supplied callbacks; plus the exchange-list runner every engine uses.
#include "comm.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>

#include "host.hpp"

namespace vinf {

int guarded_call(const std::function<void()>& f);

std::vector<vinf_xfer> matching_order(const std::vector<vinf_xfer>& xs) {
    std::vector<vinf_xfer> v = xs;
    std::stable_sort(v.begin(), v.end(), [](const vinf_xfer& a, const vinf_xfer& b) {
        return std::tie(a.peer, a.tag, a.send) < std::tie(b.peer, b.tag, b.send);
    });
    return v;
}

void run_exchange(vinf_comm* comm, const std::vector<vinf_xfer>& xs, uint8_t* base, cudaStream_t s) {
    if (xs.empty()) return;
    comm->group_start();
    for (const vinf_xfer& x : xs) {
        if (x.peer >= comm->nranks || x.peer == comm->rank)
            protocol_error("exchange peer " + std::to_string(x.peer) + " invalid for rank " +
                           std::to_string(comm->rank) + " of " + std::to_string(comm->nranks));
        if (x.send)
            comm->send(x.peer, x.tag, base + x.offset, x.bytes, s);
        else
            comm->recv(x.peer, x.tag, base + x.offset, x.bytes, s);
    }
    comm->group_end(s);
}

namespace {

// ---- NCCL (resolved at run time) ------------------------------------------------------

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
    std::string err;

    NcclApi() {
        // the NCCL torch already loaded (same library as its process group), else the system's
        const char* env = getenv("VINF_NCCL_LIB");
        if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            err = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
            return;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn && err.empty()) err = std::string("libnccl lacks ") + name;
        };
        sym(GetUniqueId, "ncclGetUniqueId");
        sym(CommInitRank, "ncclCommInitRank");
        sym(CommDestroy, "ncclCommDestroy");
        sym(GroupStart, "ncclGroupStart");
        sym(GroupEnd, "ncclGroupEnd");
        sym(Send, "ncclSend");
        sym(Recv, "ncclRecv");
        sym(AllReduce, "ncclAllReduce");
        sym(GetErrorString, "ncclGetErrorString");
        sym(GetVersion, "ncclGetVersion");
    }
    void need() const {
        if (!err.empty()) protocol_error(err);
    }
    void check(ncclResult_t r, const char* what) const {
        if (r != ncclSuccess)
            protocol_error(std::string("NCCL ") + what + ": " + (GetErrorString ? GetErrorString(r) : "error"));
    }
};

NcclApi& nccl() {
    static NcclApi api;
    return api;
}

struct NcclComm final : vinf_comm {
    ncclComm_t c = nullptr;
    const char* kind() const override { return "nccl"; }
    bool capturable() const override { return true; }
    ~NcclComm() override {
        if (c) nccl().CommDestroy(c);
    }
    void group_start() override { nccl().check(nccl().GroupStart(), "group start"); }
    void send(uint32_t peer, uint32_t, const void* p, uint64_t bytes, cudaStream_t s) override {
        nccl().check(nccl().Send(p, size_t(bytes), ncclUint8, int(peer), c, s), "send");
        bytes_sent += bytes;
        messages_sent += 1;
    }
    void recv(uint32_t peer, uint32_t, void* p, uint64_t bytes, cudaStream_t s) override {
        nccl().check(nccl().Recv(p, size_t(bytes), ncclUint8, int(peer), c, s), "recv");
    }
    void group_end(cudaStream_t) override { nccl().check(nccl().GroupEnd(), "group end"); }
    void allreduce_sum_f64(double* p, uint64_t n, cudaStream_t s) override {
        if (nranks == 1) return;
        nccl().check(nccl().AllReduce(p, p, size_t(n), ncclFloat64, ncclSum, c, s), "all-reduce");
    }
};

// ---- callbacks ---------------------------------------------------------------------------

struct OpsComm final : vinf_comm {
    vinf_transport_ops ops{};
    const char* kind() const override { return "ops"; }
    void rc(int r, const char* what) const {
        if (r != 0) protocol_error(std::string("transport callback ") + what + " failed (" + std::to_string(r) + ")");
    }
    void group_start() override {
        if (ops.group_start) rc(ops.group_start(ops.ctx), "group_start");
    }
    void send(uint32_t peer, uint32_t tag, const void* p, uint64_t bytes, cudaStream_t s) override {
        rc(ops.send(ops.ctx, peer, tag, p, bytes, s), "send");
        bytes_sent += bytes;
        messages_sent += 1;
    }
    void recv(uint32_t peer, uint32_t tag, void* p, uint64_t bytes, cudaStream_t s) override {
        rc(ops.recv(ops.ctx, peer, tag, p, bytes, s), "recv");
    }
    void group_end(cudaStream_t s) override {
        if (ops.group_end) rc(ops.group_end(ops.ctx, s), "group_end");
    }
    void allreduce_sum_f64(double* p, uint64_t n, cudaStream_t s) override {
        if (nranks == 1) return;
        rc(ops.allreduce_sum_f64(ops.ctx, p, n, s), "allreduce_sum_f64");
    }
};

// ---- in-process workers ------------------------------------------------------------------

struct LocalHub {
    explicit LocalHub(uint32_t n) : n(n), red(n) {}
    uint32_t n;
    std::mutex m;
    std::condition_variable cv;
    bool aborted = false;
    struct Post {
        const void* src = nullptr;
        uint64_t bytes = 0;
        cudaEvent_t ready = nullptr;     // sender: source complete
        cudaEvent_t consumed = nullptr;  // receiver: copy complete
        bool copied = false;
    };
    std::map<std::tuple<uint32_t, uint32_t, uint32_t>, Post> posts;  // (from, to, tag)
    std::vector<std::vector<double>> red;
    std::vector<double> result;
    uint32_t arrived = 0;
    uint64_t gen = 0;

    template <class Pred>
    void wait(std::unique_lock<std::mutex>& lk, Pred p) {
        cv.wait(lk, [&] { return aborted || p(); });
        if (aborted) protocol_error("in-process transport aborted (another worker failed)");
    }
    void abort() {
        std::lock_guard<std::mutex> g(m);
        aborted = true;
        cv.notify_all();
    }
};

void ck(cudaError_t e, const char* what) { cuda_check(int(e), what); }

struct LocalComm final : vinf_comm {
    std::shared_ptr<LocalHub> hub;
    struct Pending { uint32_t peer, tag; const void* src; void* dst; uint64_t bytes; bool send; };
    std::vector<Pending> pend;
    bool in_group = false;
    const char* kind() const override { return "local"; }
    void abort() override {
        if (hub) hub->abort();
    }
    ~LocalComm() override {
        // a worker leaving early must not strand its peers
        if (hub) hub->abort();
    }
    void group_start() override { in_group = true; }
    void send(uint32_t peer, uint32_t tag, const void* p, uint64_t bytes, cudaStream_t s) override {
        pend.push_back({peer, tag, p, nullptr, bytes, true});
        bytes_sent += bytes;
        messages_sent += 1;
        if (!in_group) group_end(s);
    }
    void recv(uint32_t peer, uint32_t tag, void* p, uint64_t bytes, cudaStream_t s) override {
        pend.push_back({peer, tag, nullptr, p, bytes, false});
        if (!in_group) group_end(s);
    }
    void group_end(cudaStream_t s) override {
        in_group = false;
        std::vector<Pending> ps;
        ps.swap(pend);
        LocalHub& H = *hub;
        // 1. publish every send (its source is complete at this point of `s`)
        for (const Pending& p : ps) {
            if (!p.send) continue;
            LocalHub::Post post;
            post.src = p.src;
            post.bytes = p.bytes;
            ck(cudaEventCreateWithFlags(&post.ready, cudaEventDisableTiming), "event");
            ck(cudaEventRecord(post.ready, s), "event record");
            std::lock_guard<std::mutex> g(H.m);
            if (!H.posts.emplace(std::make_tuple(rank, p.peer, p.tag), post).second)
                protocol_error("duplicate message tag " + std::to_string(p.tag));
            H.cv.notify_all();
        }
        // 2. receives: wait for the peer's post, copy after its source is ready
        for (const Pending& p : ps) {
            if (p.send) continue;
            const auto key = std::make_tuple(p.peer, rank, p.tag);
            std::unique_lock<std::mutex> lk(H.m);
            H.wait(lk, [&] { return H.posts.count(key) != 0; });
            LocalHub::Post& post = H.posts[key];
            if (post.bytes != p.bytes) protocol_error("context payload has wrong size");
            const void* src = post.src;
            cudaEvent_t ready = post.ready;
            lk.unlock();
            ck(cudaStreamWaitEvent(s, ready, 0), "wait ready");
            ck(cudaMemcpyAsync(p.dst, src, p.bytes, cudaMemcpyDefault, s), "exchange copy");
            cudaEvent_t done = nullptr;
            ck(cudaEventCreateWithFlags(&done, cudaEventDisableTiming), "event");
            ck(cudaEventRecord(done, s), "event record");
            lk.lock();
            LocalHub::Post& q = H.posts[key];
            q.consumed = done;
            q.copied = true;
            H.cv.notify_all();
        }
        // 3. sends: the source may be overwritten only after the receiver's copy
        for (const Pending& p : ps) {
            if (!p.send) continue;
            const auto key = std::make_tuple(rank, p.peer, p.tag);
            std::unique_lock<std::mutex> lk(H.m);
            H.wait(lk, [&] { return H.posts[key].copied; });
            LocalHub::Post post = H.posts[key];
            H.posts.erase(key);
            lk.unlock();
            ck(cudaStreamWaitEvent(s, post.consumed, 0), "wait consumed");
            cudaEventDestroy(post.consumed);
            cudaEventDestroy(post.ready);
        }
    }
    void allreduce_sum_f64(double* p, uint64_t n, cudaStream_t s) override {
        if (nranks == 1) return;
        LocalHub& H = *hub;
        std::vector<double> mine(n);
        ck(cudaMemcpyAsync(mine.data(), p, n * 8, cudaMemcpyDefault, s), "all-reduce copy");
        ck(cudaStreamSynchronize(s), "all-reduce sync");
        std::unique_lock<std::mutex> lk(H.m);
        H.red[rank] = std::move(mine);
        const uint64_t g = H.gen;
        if (++H.arrived == H.n) {
            H.result.assign(n, 0.0);
            for (uint32_t r = 0; r < H.n; ++r)  // worker order: identical bits on every rank
                for (uint64_t i = 0; i < n; ++i) H.result[i] = r == 0 ? H.red[r][i] : H.result[i] + H.red[r][i];
            H.arrived = 0;
            ++H.gen;
            H.cv.notify_all();
        } else {
            H.wait(lk, [&] { return H.gen != g; });
        }
        std::vector<double> res = H.result;
        lk.unlock();
        ck(cudaMemcpyAsync(p, res.data(), n * 8, cudaMemcpyDefault, s), "all-reduce copy");
        ck(cudaStreamSynchronize(s), "all-reduce sync");
    }
};

}  // namespace
}  // namespace vinf

using namespace vinf;

extern "C" {

int vinf_comm_nccl_unique_id(uint8_t id[128]) {
    return guarded_call([&] {
        if (!id) shape_error("null id buffer");
        nccl().need();
        ncclUniqueId u;
        nccl().check(nccl().GetUniqueId(&u), "get unique id");
        static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
        std::memcpy(id, &u, 128);
    });
}

int vinf_comm_create_nccl(const uint8_t id[128], uint32_t nranks, uint32_t rank, vinf_comm** out) {
    return guarded_call([&] {
        if (!id || !out) shape_error("null argument");
        if (nranks == 0 || rank >= nranks) range_error("rank out of range");
        nccl().need();
        ncclUniqueId u;
        std::memcpy(&u, id, 128);
        auto c = std::make_unique<NcclComm>();
        c->nranks = nranks;
        c->rank = rank;
        nccl().check(nccl().CommInitRank(&c->c, int(nranks), u, int(rank)), "comm init");
        *out = c.release();
    });
}

int vinf_comm_create_ops(const vinf_transport_ops* ops, uint32_t nranks, uint32_t rank, vinf_comm** out) {
    return guarded_call([&] {
        if (!ops || !out) shape_error("null argument");
        if (!ops->send || !ops->recv || !ops->allreduce_sum_f64) shape_error("transport ops need send, recv, allreduce");
        if (nranks == 0 || rank >= nranks) range_error("rank out of range");
        auto c = std::make_unique<OpsComm>();
        c->ops = *ops;
        c->nranks = nranks;
        c->rank = rank;
        *out = c.release();
    });
}

int vinf_comm_create_local(uint32_t nranks, vinf_comm** out) {
    return guarded_call([&] {
        if (!out) shape_error("null argument");
        if (nranks == 0) range_error("need at least one worker");
        auto hub = std::make_shared<LocalHub>(nranks);
        std::vector<std::unique_ptr<LocalComm>> cs;
        for (uint32_t r = 0; r < nranks; ++r) {
            cs.push_back(std::make_unique<LocalComm>());
            cs.back()->hub = hub;
            cs.back()->nranks = nranks;
            cs.back()->rank = r;
        }
        for (uint32_t r = 0; r < nranks; ++r) out[r] = cs[r].release();
    });
}

void vinf_comm_destroy(vinf_comm* c) { delete c; }

void vinf_comm_abort(vinf_comm* c) {
    if (c) c->abort();
}

int vinf_comm_info(const vinf_comm* c, uint32_t* nranks, uint32_t* rank, uint64_t* bytes_sent,
                   uint64_t* messages_sent) {
    return guarded_call([&] {
        if (!c) shape_error("null comm");
        if (nranks) *nranks = c->nranks;
        if (rank) *rank = c->rank;
        if (bytes_sent) *bytes_sent = c->bytes_sent;
        if (messages_sent) *messages_sent = c->messages_sent;
    });
}

int vinf_comm_allreduce_sum_f64(vinf_comm* c, double* p, uint64_t n, void* stream) {
    return guarded_call([&] {
        if (!c || (!p && n)) shape_error("null argument");
        c->allreduce_sum_f64(p, n, static_cast<cudaStream_t>(stream));
    });
}

}  // extern "C"
