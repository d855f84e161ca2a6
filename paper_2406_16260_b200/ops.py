"""Temporal-module operators on CUDA tensors, mirroring the reference C++ API
(/root/reference/proj/src/core/ops.hpp:49-124) name for name. Every call goes through
the C ABI of libvinf_b200.so (hand-written sm_100a kernels); torch only supplies device
memory and the current stream.

Tensors are torch CUDA tensors of shape [F, H, W, C] (contiguous, channels innermost,
tensor.hpp:13-24), dtype float32 (fp32 mode, bf16x3 tensor-core GEMMs) or bfloat16.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import ConfigError, ProtocolError, ShapeError, TransportError, VinfError  # noqa: F401

_DT = {torch.float32: _lib.VINF_F32, torch.bfloat16: _lib.VINF_BF16}


def _L():
    return _lib.load()


def _stream(t: torch.Tensor | None = None):
    dev = t.device if t is not None else torch.device("cuda")
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _ten(x: torch.Tensor | None) -> _lib.Tensor | None:
    if x is None or x.numel() == 0:
        return None
    if not x.is_cuda:
        raise ShapeError("tensor must live on a CUDA device")
    if x.dim() != 4:
        raise ShapeError(f"expected [F,H,W,C], got shape {tuple(x.shape)}")
    if x.dtype not in _DT:
        raise ShapeError(f"unsupported dtype {x.dtype}")
    if not x.is_contiguous():
        raise ShapeError("tensor must be contiguous")
    f, h, w, c = x.shape
    return _lib.Tensor(x.data_ptr(), f, h, w, c, _DT[x.dtype])


def _ref(t: _lib.Tensor | None):
    return C.byref(t) if t is not None else None


# ---- token sets / seeds (integer exact) -----------------------------------------


def build_local_window(a: int, frames: int, n_local: int) -> list[int]:
    """ops.cpp:177-186"""
    out = (C.c_uint32 * (n_local + 2))()
    n = C.c_uint32()
    _lib.check(_L().vinf_build_local_window(a, frames, n_local, out, n_local + 2, C.byref(n)))
    return list(out[: n.value])


def build_global_index_set(frames: int, n_global: int) -> list[int]:
    """ops.cpp:188-198"""
    cap = max(n_global, 1)
    out = (C.c_uint32 * cap)()
    n = C.c_uint32()
    _lib.check(_L().vinf_build_global_index_set(frames, n_global, out, cap, C.byref(n)))
    return list(out[: n.value])


def mix_seed(seed: int, salt: int) -> int:
    """rng.hpp:34-37"""
    return int(_L().vinf_mix_seed(seed, salt))


def tensor_from_seed(dims, seed: int, first_elem: int = 0, dtype=torch.float32, device=None,
                     scale: float = 1.0) -> torch.Tensor:
    """tensor_from_seed_at (tensor.cpp:98-106), generated on the device bit-exactly."""
    device = device or torch.device("cuda")
    out = torch.empty(tuple(dims), dtype=dtype, device=device)
    _lib.check(_L().vinf_fill_seeded(C.c_void_p(out.data_ptr()), _DT[dtype], out.numel(), seed,
                                     first_elem, C.c_float(scale), _stream(out)))
    return out


# ---- parameter bundles ----------------------------------------------------------


class ConvKernel:
    """ConvKernel (ops.hpp:14-21): weights [taps][out][in], bias [C], fp32 on device."""

    def __init__(self, taps: int, weights: torch.Tensor, bias: torch.Tensor):
        weights = weights.detach().to(torch.float32).contiguous()
        bias = bias.detach().to(torch.float32).contiguous()
        C_ = bias.numel()
        if weights.numel() != taps * C_ * C_:
            raise ShapeError("conv kernel sized for wrong channel count")
        self.taps, self.C = taps, C_
        self.weights, self.bias = weights, bias
        h = C.c_void_p()
        _lib.check(_L().vinf_conv_kernel_create(taps, C_, C.c_void_p(weights.data_ptr()),
                                                C.c_void_p(bias.data_ptr()), C.byref(h)))
        self._h = h

    def channels(self) -> int:
        return self.C

    def halo(self) -> int:
        return (self.taps - 1) // 2

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None and _lib._lib is not None:
            _lib._lib.vinf_conv_kernel_destroy(self._h)
            self._h = None


class AttentionParams:
    """AttentionParams (ops.hpp:32-36); `heads` is an extension (1 = the reference)."""

    def __init__(self, dim: int, wq, wk, wv, wo, scale: float | None = None, heads: int = 1):
        ws = [w.detach().to(torch.float32).contiguous() for w in (wq, wk, wv, wo)]
        for w in ws:
            if w.numel() != dim * dim:
                raise ShapeError("attention projections must be C x C")
        if scale is None:
            scale = float(np.float32(1.0) / np.sqrt(np.float32(dim // heads)))
        self.dim, self.heads, self.scale = dim, heads, scale
        self._w = ws
        h = C.c_void_p()
        _lib.check(_L().vinf_attention_params_create(dim, heads, C.c_float(scale),
                                                     *[C.c_void_p(w.data_ptr()) for w in ws],
                                                     C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None and _lib._lib is not None:
            _lib._lib.vinf_attention_params_destroy(self._h)
            self._h = None


@dataclass
class GroupNormParams:
    """GroupNormParams (ops.hpp:23-30)."""
    groups: int
    gamma: torch.Tensor
    beta: torch.Tensor
    epsilon: float = 1e-5

    def _c(self):
        self._g = self.gamma.detach().to(torch.float32).contiguous()
        self._b = self.beta.detach().to(torch.float32).contiguous()
        return _lib.GroupNormParams(self.groups, self._g.data_ptr(), self._b.data_ptr(),
                                    self.epsilon)


@dataclass
class DualScopeConfig:
    """DualScopeConfig (ops.hpp:38-43)."""
    n_local: int = 16
    n_global: int = 16
    bias: float = 10.0
    t_star: float = 800.0

    def _c(self):
        return _lib.DualScopeConfig(self.n_local, self.n_global, self.bias, self.t_star)


# ---- operators --------------------------------------------------------------------


def _like(v: torch.Tensor, frames: int | None = None, dtype=None) -> torch.Tensor:
    shape = (frames if frames is not None else v.shape[0],) + tuple(v.shape[1:])
    return torch.empty(shape, dtype=dtype or v.dtype, device=v.device)


def spatial_affine_tanh(v: torch.Tensor, a: torch.Tensor, c: torch.Tensor) -> torch.Tensor:
    """ops.cpp:42-55"""
    out = _like(v)
    a = a.detach().to(torch.float32).contiguous()
    c = c.detach().to(torch.float32).contiguous()
    _lib.check(_L().vinf_spatial_affine_tanh(_ref(_ten(v)), C.c_void_p(a.data_ptr()),
                                             C.c_void_p(c.data_ptr()), _ref(_ten(out)), _stream(v)))
    return out


def conv_over_extended(ext: torch.Tensor, out_start: int, out_len: int,
                       kern: ConvKernel) -> torch.Tensor:
    """ops.cpp:73-104"""
    if out_len == 0 or out_start > ext.shape[0] or out_len > ext.shape[0] - out_start:
        raise ShapeError("conv output range outside extended tensor")
    out = _like(ext, out_len)
    _lib.check(_L().vinf_conv_over_extended(_ref(_ten(ext)), out_start, out_len, kern._h,
                                            _ref(_ten(out)), _stream(ext)))
    return out


def temporal_conv(v: torch.Tensor, kern: ConvKernel) -> torch.Tensor:
    """ops.cpp:106-108"""
    out = _like(v)
    _lib.check(_L().vinf_temporal_conv(_ref(_ten(v)), kern._h, _ref(_ten(out)), _stream(v)))
    return out


def group_means(v: torch.Tensor, groups: int) -> torch.Tensor:
    """ops.cpp:112-123 -> f64 device tensor [groups]"""
    out = torch.empty(groups, dtype=torch.float64, device=v.device)
    _lib.check(_L().vinf_group_means(_ref(_ten(v)), groups, C.c_void_p(out.data_ptr()), _stream(v)))
    return out


def group_sqdev(v: torch.Tensor, groups: int, means: torch.Tensor) -> torch.Tensor:
    """ops.cpp:125-142"""
    means = means.to(device=v.device, dtype=torch.float64).contiguous()
    if means.numel() != groups:
        raise ShapeError("means must have one entry per group")
    out = torch.empty(groups, dtype=torch.float64, device=v.device)
    _lib.check(_L().vinf_group_sqdev(_ref(_ten(v)), groups, C.c_void_p(means.data_ptr()),
                                     C.c_void_p(out.data_ptr()), _stream(v)))
    return out


def group_partial_sums(v: torch.Tensor, groups: int, center: torch.Tensor | None = None):
    """Per-clip sum (or sum of squared deviations about `center`) per group, f64."""
    out = torch.empty(groups, dtype=torch.float64, device=v.device)
    cptr = None
    if center is not None:
        center = center.to(device=v.device, dtype=torch.float64).contiguous()
        cptr = C.c_void_p(center.data_ptr())
    _lib.check(_L().vinf_group_partial_sums(_ref(_ten(v)), groups, cptr,
                                            C.c_void_p(out.data_ptr()), _stream(v)))
    return out


def normalize_with_stats(v: torch.Tensor, p: GroupNormParams, means: torch.Tensor,
                         vars_: torch.Tensor) -> torch.Tensor:
    """ops.cpp:144-167"""
    means = means.to(device=v.device, dtype=torch.float64).contiguous()
    vars_ = vars_.to(device=v.device, dtype=torch.float64).contiguous()
    if means.numel() != p.groups or vars_.numel() != p.groups:
        raise ShapeError("stats must have one entry per group")
    out = _like(v)
    cp = p._c()
    _lib.check(_L().vinf_normalize_with_stats(_ref(_ten(v)), C.byref(cp),
                                              C.c_void_p(means.data_ptr()),
                                              C.c_void_p(vars_.data_ptr()), _ref(_ten(out)),
                                              _stream(v)))
    return out


def group_norm(v: torch.Tensor, p: GroupNormParams) -> torch.Tensor:
    """ops.cpp:169-173"""
    out = _like(v)
    cp = p._c()
    _lib.check(_L().vinf_group_norm(_ref(_ten(v)), C.byref(cp), _ref(_ten(out)), _stream(v)))
    return out


def dual_scope_reference(v: torch.Tensor, t: float, p: AttentionParams,
                         cfg: DualScopeConfig) -> torch.Tensor:
    """ops.cpp:291-338 (the reference's name; this is the B200 implementation)"""
    out = _like(v)
    cc = cfg._c()
    _lib.check(_L().vinf_dual_scope_attention(_ref(_ten(v)), C.c_double(t), p._h, C.byref(cc),
                                              _ref(_ten(out)), _stream(v)))
    return out


dual_scope_attention = dual_scope_reference


def attention_full(v: torch.Tensor, p: AttentionParams) -> torch.Tensor:
    """ops.cpp:264-289"""
    out = _like(v)
    _lib.check(_L().vinf_attention_full(_ref(_ten(v)), p._h, _ref(_ten(out)), _stream(v)))
    return out

