"""Clip parallelism: frame-axis partition, the 3-step context sync and the distributed
operator forms, mirroring /root/reference/proj/src/core/clip_parallel.hpp:14-84.

Compute runs in the sm_100a kernels behind the C ABI; context moves run over a
`Transport` (transport.py). Plans and traffic closed forms are integer-exact host code
in the same library.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum

import torch

from . import _lib
from ._lib import ConfigError, ProtocolError, ShapeError  # noqa: F401
from .ops import (AttentionParams, ConvKernel, DualScopeConfig, GroupNormParams, _L, _ref,
                  _stream, _ten, build_global_index_set, group_partial_sums, normalize_with_stats)
from .transport import Msg, Transport


class LayerKind(IntEnum):  # metrics.hpp:11
    Conv = 1
    GroupNorm = 2
    Attention = 3


@dataclass
class FrameRange:
    start: int
    len: int


@dataclass
class ClipPlan:
    """clip_parallel.hpp:14-19: worker i owns frames [i*f_clip, (i+1)*f_clip)."""
    n: int
    f: int
    f_clip: int
    ranges: list = field(default_factory=list)


def make_plan(frames: int, workers: int) -> ClipPlan:
    """clip_parallel.cpp:54-67"""
    fc = C.c_uint32()
    _lib.check(_L().vinf_make_plan(frames, workers, C.byref(fc)))
    return ClipPlan(workers, frames, fc.value,
                    [FrameRange(i * fc.value, fc.value) for i in range(workers)])


def partition(x: torch.Tensor, workers: int) -> list[torch.Tensor]:
    """clip_parallel.cpp:69-76 (views; frame slicing is contiguous)."""
    plan = make_plan(x.shape[0], workers)
    return [x[r.start:r.start + r.len] for r in plan.ranges]


@dataclass
class LayerHaloSpec:
    """clip_parallel.hpp:28-32"""
    kind: LayerKind = LayerKind.Conv
    halo: int = 0
    global_frames: int = 0


@dataclass
class TemporalContext:
    """clip_parallel.hpp:40-44; None at the video edge / when not synchronised."""
    c_pre: torch.Tensor | None = None
    c_post: torch.Tensor | None = None
    c_global: torch.Tensor | None = None


def global_members_in_range(frames: int, n_global: int, r: FrameRange) -> list[int]:
    """clip_parallel.cpp:85-91"""
    cap = max(n_global, 1)
    out = (C.c_uint32 * cap)()
    n = C.c_uint32()
    _lib.check(_L().vinf_global_members_in_range(frames, n_global, r.start, r.len, out, cap,
                                                 C.byref(n)))
    return list(out[: n.value])


@dataclass
class TrafficPrediction:
    bytes_sent: int = 0
    bytes_contributed: int = 0
    messages: int = 0


def predict_sync_traffic(plan: ClipPlan, spec: LayerHaloSpec, worker: int,
                         frame_bytes: int) -> TrafficPrediction:
    """clip_parallel.cpp:343-375"""
    out = (C.c_uint64 * 3)()
    _lib.check(_L().vinf_predict_sync_traffic(plan.f, plan.n, spec.halo, spec.global_frames,
                                              worker, frame_bytes, out))
    return TrafficPrediction(*out)


def predict_groupnorm_traffic(plan: ClipPlan, groups: int, worker: int) -> TrafficPrediction:
    """clip_parallel.cpp:377-387"""
    out = (C.c_uint64 * 3)()
    _lib.check(_L().vinf_predict_groupnorm_traffic(plan.f, plan.n, groups, worker, out))
    return TrafficPrediction(*out)


def sync_contexts(t: Transport, plan: ClipPlan, spec: LayerHaloSpec, v_in: torch.Tensor,
                  ablate: bool = False) -> TemporalContext:
    """clip_parallel.cpp:93-192. T1 gathers every worker's members of the global index set
    (in worker order = global-index order); T2/T3 swap `halo` boundary frames with both
    neighbours. All messages of one call go out as one batch. ablate=True returns
    zero-filled contexts of the right shape and moves nothing."""
    i, n = t.rank, plan.n
    if t.world != n:
        raise _lib.TransportError("transport world does not match clip plan")
    if v_in.shape[0] != plan.f_clip:
        raise ProtocolError(f"worker {i} clip has {v_in.shape[0]} frames, plan says {plan.f_clip}")
    if spec.halo > plan.f_clip:
        raise ConfigError(f"halo of {spec.halo} frames exceeds clip size {plan.f_clip}")
    frame_shape = tuple(v_in.shape[1:])
    ctx = TemporalContext()
    msgs: list[Msg] = []
    if spec.global_frames > 0:
        members = [global_members_in_range(plan.f, spec.global_frames, r) for r in plan.ranges]
        ctx.c_global = torch.zeros((spec.global_frames,) + frame_shape, dtype=v_in.dtype,
                                   device=v_in.device)
        if not ablate:
            slot = 0
            for w in range(n):
                for k, lf in enumerate(members[w]):
                    dst = ctx.c_global[slot]
                    if w == i:
                        dst.copy_(v_in[lf])
                    else:
                        msgs.append(Msg(w, False, dst, 100000 + slot))
                    slot += 1
            # our own members go to every other worker
            base = sum(len(members[w]) for w in range(i))
            for k, lf in enumerate(members[i]):
                for w in range(n):
                    if w != i:
                        msgs.append(Msg(w, True, v_in[lf], 100000 + base + k))
    if spec.halo > 0 and n > 1:
        h = spec.halo
        if i > 0:
            ctx.c_pre = torch.zeros((h,) + frame_shape, dtype=v_in.dtype, device=v_in.device)
        if i + 1 < n:
            ctx.c_post = torch.zeros((h,) + frame_shape, dtype=v_in.dtype, device=v_in.device)
        if not ablate:
            if i + 1 < n:  # HaloFwd: last h frames -> next worker's c_pre; its first h -> c_post
                msgs.append(Msg(i + 1, True, v_in[plan.f_clip - h:], 0))
                msgs.append(Msg(i + 1, False, ctx.c_post, 1))
            if i > 0:
                msgs.append(Msg(i - 1, False, ctx.c_pre, 0))
                msgs.append(Msg(i - 1, True, v_in[:h], 1))
    if msgs:
        t.exchange(msgs)
    return ctx


def conv_parallel(plan: ClipPlan, worker: int, v: torch.Tensor, ctx: TemporalContext,
                  kern: ConvKernel) -> torch.Tensor:
    """clip_parallel.cpp:194-209"""
    out = torch.empty_like(v)
    _lib.check(_L().vinf_conv_parallel(plan.f, plan.n, worker, _ref(_ten(v)),
                                       _ref(_ten(ctx.c_pre)), _ref(_ten(ctx.c_post)), kern._h,
                                       _ref(_ten(out)), _stream(v)))
    return out


def group_norm_parallel(t: Transport, plan: ClipPlan, v: torch.Tensor, p: GroupNormParams,
                        ablate: bool = False) -> torch.Tensor:
    """clip_parallel.cpp:211-254: round 1 combines per-clip means, round 2 the squared
    deviations about the global mean (equal clip sizes make both plain averages exact).
    Partial sums are f64 and combined with one all-reduce per round."""
    count = v.numel() // p.groups  # per clip
    s1 = group_partial_sums(v, p.groups)
    if ablate:
        mean = s1 / count
        var = group_partial_sums(v, p.groups, mean) / count
        return normalize_with_stats(v, p, mean, var)
    t.allreduce_sum_(s1)
    mean = s1 / (count * plan.n)
    s2 = group_partial_sums(v, p.groups, mean)
    t.allreduce_sum_(s2)
    var = s2 / (count * plan.n)
    return normalize_with_stats(v, p, mean, var)


def attention_parallel(plan: ClipPlan, worker: int, v: torch.Tensor, ctx: TemporalContext,
                       t: float, p: AttentionParams, cfg: DualScopeConfig) -> torch.Tensor:
    """clip_parallel.cpp:256-341"""
    out = torch.empty_like(v)
    cc = cfg._c()
    _lib.check(_L().vinf_attention_parallel(plan.f, plan.n, worker, _ref(_ten(v)),
                                            _ref(_ten(ctx.c_pre)), _ref(_ten(ctx.c_post)),
                                            _ref(_ten(ctx.c_global)), C.c_double(t), p._h,
                                            C.byref(cc), _ref(_ten(out)), _stream(v)))
    return out
