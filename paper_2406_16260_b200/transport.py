"""Transports for the clip-parallel context sync (the reference's Transport,
transport.hpp:20-43, re-based on torch.distributed).

`Transport` is the per-worker view the reference's SPMD code takes: point-to-point
messages matched by (peer, tag) plus a sum all-reduce. Two backends:

* `DistTransport` — one process per GPU over torch.distributed (NCCL on B200, gloo
  on CPU hosts for tests). All point-to-point messages of one exchange go out as one
  `batch_isend_irecv` group, so NVSwitch carries both halo directions and the global
  frames concurrently (no even/odd pair staging needed).
* `LocalHub` / `LocalTransport` — N workers as threads of one process (the shape of
  the reference's run_inproc_workers, transport_inproc.cpp:148-189); messages are
  device-to-device copies matched at a rendezvous.
"""
from __future__ import annotations

import threading
from dataclasses import dataclass

import torch


@dataclass
class Msg:
    peer: int
    send: bool
    tensor: torch.Tensor  # send: source; recv: destination (same numel/dtype)
    tag: int


class Transport:
    rank: int
    world: int
    bytes_sent: int = 0
    messages_sent: int = 0

    def exchange(self, msgs: list[Msg]) -> None:
        raise NotImplementedError

    def allreduce_sum_(self, t: torch.Tensor) -> None:
        raise NotImplementedError

    def _count(self, msgs: list[Msg]) -> None:
        for m in msgs:
            if m.send:
                self.bytes_sent += m.tensor.numel() * m.tensor.element_size()
                self.messages_sent += 1


class DistTransport(Transport):
    """torch.distributed point-to-point + all-reduce on the default process group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.bytes_sent = 0
        self.messages_sent = 0

    def exchange(self, msgs: list[Msg]) -> None:
        if not msgs:
            return
        d = self.dist
        # Both ends list a pair's messages in the same (peer, tag) order, which is the
        # order NCCL matches them in.
        ordered = sorted(msgs, key=lambda m: (m.peer, m.tag, m.send))
        ops = []
        for m in ordered:
            fn = d.isend if m.send else d.irecv
            ops.append(d.P2POp(fn, m.tensor, m.peer, self.group, m.tag))
        for w in d.batch_isend_irecv(ops):
            w.wait()
        self._count(msgs)

    def allreduce_sum_(self, t: torch.Tensor) -> None:
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)


class LocalHub:
    """In-process rendezvous for N worker threads (strict: every exchange is a barrier)."""

    def __init__(self, world: int):
        self.world = world
        self._barrier = threading.Barrier(world)
        self._posted: list[list[Msg] | None] = [None] * world
        self._red: list[torch.Tensor | None] = [None] * world

    def transport(self, rank: int) -> "LocalTransport":
        return LocalTransport(self, rank)

    def abort(self) -> None:
        self._barrier.abort()


class LocalTransport(Transport):
    def __init__(self, hub: LocalHub, rank: int):
        self.hub, self.rank, self.world = hub, rank, hub.world
        self.bytes_sent = 0
        self.messages_sent = 0

    def exchange(self, msgs: list[Msg]) -> None:
        hub = self.hub
        hub._posted[self.rank] = msgs
        hub._barrier.wait()
        for m in msgs:
            if m.send:
                continue
            src = [s for s in hub._posted[m.peer] if s.send and s.peer == self.rank and s.tag == m.tag]
            if len(src) != 1:
                from ._lib import ProtocolError
                raise ProtocolError(f"worker {self.rank}: no unique message from {m.peer} tag {m.tag}")
            s = src[0]
            if s.tensor.numel() != m.tensor.numel():
                from ._lib import ProtocolError
                raise ProtocolError("context payload has wrong size")
            m.tensor.copy_(s.tensor.view(m.tensor.dtype).reshape(m.tensor.shape))
        hub._barrier.wait()
        self._count(msgs)

    def allreduce_sum_(self, t: torch.Tensor) -> None:
        hub = self.hub
        hub._red[self.rank] = t.clone()
        hub._barrier.wait()
        total = hub._red[0].clone()
        for r in range(1, self.world):  # fixed worker order: identical on every rank
            total += hub._red[r]
        hub._barrier.wait()
        t.copy_(total)


def run_local_workers(n: int, body) -> list:
    """Runs body(transport) on n threads over a fresh LocalHub; rethrows the first failure
    (transport_inproc.cpp:148-189)."""
    hub = LocalHub(n)
    results: list = [None] * n
    errors: list = []

    def work(r):
        try:
            results[r] = body(hub.transport(r))
        except BaseException as e:  # noqa: BLE001
            errors.append(e)
            hub.abort()

    threads = [threading.Thread(target=work, args=(r,)) for r in range(n)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    real = [e for e in errors if not isinstance(e, threading.BrokenBarrierError)]
    if real or errors:
        raise (real or errors)[0]
    return results
