"""Communicators of the C++ clip-parallel executor (include/vinf_temporal.h, csrc/comm.cpp):
the reference's Transport (transport.hpp:20-43) for the device engine.

    comm = NcclComm.create()          # one process per GPU, after torch.distributed init
    comms = local_comms(n)            # n in-process workers (threads), e.g. n clips on one GPU
    comm = OpsComm(GlooPointerTransport())   # callbacks: any transport (CPU tests: gloo)

The exchanges themselves (which byte ranges go where, in which order) are the C++
layout's plan; these objects only move bytes.
"""
from __future__ import annotations

import ctypes as C

from . import _lib


class Comm:
    """Owns one vinf_comm handle."""

    def __init__(self, handle: C.c_void_p, keep=None):
        self._h = handle
        self._keep = keep  # callback objects the C side points at

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def info(self) -> dict:
        n, r = C.c_uint32(), C.c_uint32()
        b, m = C.c_uint64(), C.c_uint64()
        _lib.check(_lib.load().vinf_comm_info(self._h, C.byref(n), C.byref(r), C.byref(b), C.byref(m)))
        return {"nranks": n.value, "rank": r.value, "bytes_sent": b.value, "messages_sent": m.value}

    def allreduce_sum_f64(self, ptr: int, count: int, stream: int = 0) -> None:
        _lib.check(_lib.load().vinf_comm_allreduce_sum_f64(self._h, C.c_void_p(ptr), count, C.c_void_p(stream)))

    def abort(self) -> None:
        if self._h:
            _lib.load().vinf_comm_abort(self._h)

    def close(self) -> None:
        if getattr(self, "_h", None) and _lib._lib is not None:
            _lib._lib.vinf_comm_destroy(self._h)
        self._h = None

    def __del__(self):
        self.close()


class NcclComm(Comm):
    @classmethod
    def create(cls, group=None) -> "NcclComm":
        """Collective over torch.distributed's (default) group: rank 0 draws the NCCL id,
        every rank receives it and joins on its current CUDA device."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        ident = (C.c_uint8 * 128)()
        if rank == 0:
            _lib.check(_lib.load().vinf_comm_nccl_unique_id(ident))
        box = [bytes(ident)]
        dist.broadcast_object_list(box, src=0, group=group)
        ident = (C.c_uint8 * 128).from_buffer_copy(box[0])
        h = C.c_void_p()
        _lib.check(_lib.load().vinf_comm_create_nccl(ident, world, rank, C.byref(h)))
        return cls(h)


def local_comms(n: int) -> list[Comm]:
    """n communicators sharing one in-process hub (one per worker thread)."""
    arr = (C.c_void_p * n)()
    _lib.check(_lib.load().vinf_comm_create_local(n, arr))
    return [Comm(C.c_void_p(arr[i])) for i in range(n)]


class OpsComm(Comm):
    """A communicator whose messages are Python callbacks on raw pointers. `transport`
    provides send(peer, tag, ptr, nbytes), recv(peer, tag, ptr, nbytes), flush() (the
    group end) and allreduce_f64(ptr, count); rank / world attributes."""

    def __init__(self, transport):
        t = transport
        errors: list = []

        def guard(fn):
            def call(*a):
                try:
                    fn(*a)
                    return 0
                except BaseException as e:  # noqa: BLE001 - reported as a status code
                    errors.append(e)
                    return 1
            return call

        cbs = _lib.TransportOps(
            None,
            _lib.GROUP_START_FN(guard(lambda ctx: None)),
            _lib.SEND_FN(guard(lambda ctx, peer, tag, p, n, s: t.send(peer, tag, p, n))),
            _lib.RECV_FN(guard(lambda ctx, peer, tag, p, n, s: t.recv(peer, tag, p, n))),
            _lib.GROUP_END_FN(guard(lambda ctx, s: t.flush())),
            _lib.ALLREDUCE_FN(guard(lambda ctx, p, n, s: t.allreduce_f64(p, n))))
        h = C.c_void_p()
        _lib.check(_lib.load().vinf_comm_create_ops(C.byref(cbs), t.world, t.rank, C.byref(h)))
        super().__init__(h, keep=(cbs, t))
        self.errors = errors


class GlooPointerTransport:
    """torch.distributed point-to-point on HOST memory given as raw pointers (CPU hosts,
    gloo): what an OpsComm needs to drive the exchange plans without a GPU."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self._ops: list = []

    @staticmethod
    def _view(ptr: int, nbytes: int):
        import torch
        return torch.frombuffer((C.c_uint8 * nbytes).from_address(ptr), dtype=torch.uint8)

    def send(self, peer, tag, ptr, nbytes):
        self._ops.append(self.dist.P2POp(self.dist.isend, self._view(ptr, nbytes).clone(), peer, self.group, tag))

    def recv(self, peer, tag, ptr, nbytes):
        self._ops.append(self.dist.P2POp(self.dist.irecv, self._view(ptr, nbytes), peer, self.group, tag))

    def flush(self):
        ops, self._ops = self._ops, []
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()

    def allreduce_f64(self, ptr, count):
        import torch
        t = torch.frombuffer((C.c_double * count).from_address(ptr), dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
