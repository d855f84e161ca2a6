// Communicators for the clip-parallel context sync: the reference's Transport
// (transport.hpp:20-43) re-based on NVLink. One vinf_comm per worker; point-to-point
// messages matched by (peer, tag) inside a group, plus a sum all-reduce of f64.
//
//   * NCCL   : ncclSend / ncclRecv grouped per exchange, ncclAllReduce for the GroupNorm
//              sums (NVSwitch carries both halo directions and the global frames at once);
//              libnccl is resolved at run time (the one torch already loaded, else
//              libnccl.so.2), so the library has no link-time NCCL dependency.
//   * local  : N workers as threads of one process (the shape of run_inproc_workers,
//              transport_inproc.cpp:148-189): messages are device copies ordered by
//              events, the all-reduce sums in worker order on the host.
//   * ops    : caller-supplied callbacks (vinf_transport_ops), e.g. a gloo transport in
//              CPU tests driving the same exchange plans.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/vinf_temporal.h"

struct vinf_comm {
    uint32_t nranks = 1, rank = 0;
    uint64_t bytes_sent = 0, messages_sent = 0;
    virtual ~vinf_comm() = default;
    virtual const char* kind() const = 0;
    // Messages posted between group_start and group_end complete (in stream order) at
    // group_end: the receive buffers are written and the send buffers may be reused by
    // work enqueued on `stream` afterwards.
    virtual void group_start() = 0;
    virtual void send(uint32_t peer, uint32_t tag, const void* p, uint64_t bytes, cudaStream_t s) = 0;
    virtual void recv(uint32_t peer, uint32_t tag, void* p, uint64_t bytes, cudaStream_t s) = 0;
    virtual void group_end(cudaStream_t s) = 0;
    virtual void allreduce_sum_f64(double* p, uint64_t n, cudaStream_t s) = 0;
    // Whether its operations may be captured into a CUDA graph (NCCL: yes).
    virtual bool capturable() const { return false; }
    // Unblocks peers waiting on this worker (in-process transport) after a failure.
    virtual void abort() {}
};

namespace vinf {

// Runs one exchange list (vinf_layout_exchange order) over `comm` with workspace base
// `base`: every transfer in one group, posted in (peer, tag) order on both ends, which
// is the order NCCL matches point-to-point messages of a peer pair in.
void run_exchange(vinf_comm* comm, const std::vector<vinf_xfer>& xs, uint8_t* base, cudaStream_t s);
// The list sorted into that matching order (engines cache it).
std::vector<vinf_xfer> matching_order(const std::vector<vinf_xfer>& xs);

}  // namespace vinf
