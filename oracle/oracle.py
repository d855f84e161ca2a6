"""ctypes bindings for the CPU checkers — TEST INFRASTRUCTURE ONLY.

`Oracle` wraps oracle/_build/liboracle.so (the plain-C restatement, vinf_oracle.c);
`Reference` wraps oracle/_ref/libvinf_ref.so (the unmodified reference compiled
from its sources + ref_shim.cpp). Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import this module; the
product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libvinf_ref.so")

_f32p = C.POINTER(C.c_float)
_f64p = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)


def build(force: bool = False) -> None:
    """Compile the checkers (make -C oracle). Reference part only if its tree exists."""
    if force or not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    elif not os.path.exists(REF_SO) and os.path.isdir("/root/reference/proj/src/core"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _p(a: np.ndarray | None, typ):
    if a is None:
        return C.cast(None, typ)
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(typ)


def f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


class BlockParams:
    """One block's parameters in the reference layout (pipeline.hpp:30-36)."""

    def __init__(self, C: int, taps: int = 3):
        self.C, self.taps = C, taps
        self.stub_a = np.zeros(C, np.float32)
        self.stub_c = np.zeros(C, np.float32)
        self.conv_w = np.zeros(taps * C * C, np.float32)
        self.conv_b = np.zeros(C, np.float32)
        self.gamma = np.zeros(C, np.float32)
        self.beta = np.zeros(C, np.float32)
        self.wq = np.zeros(C * C, np.float32)
        self.wk = np.zeros(C * C, np.float32)
        self.wv = np.zeros(C * C, np.float32)
        self.wo = np.zeros(C * C, np.float32)

    def arrays(self):
        return [self.stub_a, self.stub_c, self.conv_w, self.conv_b, self.gamma, self.beta,
                self.wq, self.wk, self.wv, self.wo]


class Oracle:
    """The plain-C restatement (oracle/vinf_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        L.orc_mix_seed.restype = C.c_uint64
        L.orc_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_fill_seeded.argtypes = [_f32p, C.c_size_t, C.c_uint64, C.c_uint64, C.c_float]

    # --- rng / weights -----------------------------------------------------
    def fill_seeded(self, n, seed, first_elem=0, scale=1.0):
        out = np.empty(n, np.float32)
        self.lib.orc_fill_seeded(_p(out, _f32p), n, seed, first_elem, C.c_float(scale))
        return out

    def tensor_from_seed(self, dims, seed, first_elem=0):
        return self.fill_seeded(int(np.prod(dims)), seed, first_elem).reshape(dims)

    def mix_seed(self, seed, salt):
        return int(self.lib.orc_mix_seed(seed, salt))

    def build_block(self, C_, taps=3, weight_seed=1, block=0) -> BlockParams:
        bp = BlockParams(C_, taps)
        rc = self.lib.orc_build_block(C.c_uint32(C_), C.c_uint32(taps), C.c_uint64(weight_seed),
                                      C.c_uint32(block), *[_p(a, _f32p) for a in bp.arrays()])
        assert rc == 0, rc
        return bp

    # --- ops -----------------------------------------------------------------
    def spatial_affine_tanh(self, v, a, c):
        v = f32(v)
        out = np.empty_like(v)
        self.lib.orc_spatial_affine_tanh(_p(v, _f32p), C.c_size_t(v.size), C.c_uint32(v.shape[-1]),
                                         _p(f32(a), _f32p), _p(f32(c), _f32p), _p(out, _f32p))
        return out

    def conv_over_extended(self, ext, out_start, out_len, taps, w, b):
        ext = f32(ext)
        F, H, W, Cc = ext.shape
        out = np.empty((out_len, H, W, Cc), np.float32)
        rc = self.lib.orc_conv_over_extended(_p(ext, _f32p), F, H, W, Cc, out_start, out_len, taps,
                                             _p(f32(w), _f32p), _p(f32(b), _f32p), _p(out, _f32p))
        if rc:
            raise ValueError(f"orc_conv_over_extended rc={rc}")
        return out

    def temporal_conv(self, v, taps, w, b):
        return self.conv_over_extended(v, 0, v.shape[0], taps, w, b)

    def group_stats(self, v, groups):
        v = f32(v)
        m = np.empty(groups, np.float64)
        s = np.empty(groups, np.float64)
        rc = self.lib.orc_group_means(_p(v, _f32p), C.c_size_t(v.size), C.c_uint32(v.shape[-1]),
                                      C.c_uint32(groups), _p(m, _f64p))
        if rc:
            raise ValueError("groups must divide channels")
        self.lib.orc_group_sqdev(_p(v, _f32p), C.c_size_t(v.size), C.c_uint32(v.shape[-1]),
                                 C.c_uint32(groups), _p(m, _f64p), _p(s, _f64p))
        return m, s

    def group_sqdev(self, v, groups, means):
        v = f32(v)
        means = np.ascontiguousarray(means, np.float64)
        s = np.empty(groups, np.float64)
        self.lib.orc_group_sqdev(_p(v, _f32p), C.c_size_t(v.size), C.c_uint32(v.shape[-1]),
                                 C.c_uint32(groups), _p(means, _f64p), _p(s, _f64p))
        return s

    def normalize_with_stats(self, v, groups, gamma, beta, eps, means, vars_):
        v = f32(v)
        out = np.empty_like(v)
        rc = self.lib.orc_normalize_with_stats(
            _p(v, _f32p), C.c_size_t(v.size), C.c_uint32(v.shape[-1]), C.c_uint32(groups),
            _p(f32(gamma), _f32p), _p(f32(beta), _f32p), C.c_float(eps),
            _p(np.ascontiguousarray(means, np.float64), _f64p),
            _p(np.ascontiguousarray(vars_, np.float64), _f64p), _p(out, _f32p))
        if rc:
            raise ValueError(f"normalize rc={rc}")
        return out

    def group_norm(self, v, groups, gamma, beta, eps=1e-5):
        v = f32(v)
        out = np.empty_like(v)
        rc = self.lib.orc_group_norm(_p(v, _f32p), C.c_size_t(v.size), C.c_uint32(v.shape[-1]),
                                     C.c_uint32(groups), _p(f32(gamma), _f32p),
                                     _p(f32(beta), _f32p), C.c_float(eps), _p(out, _f32p))
        if rc:
            raise ValueError(f"group_norm rc={rc}")
        return out

    def build_local_window(self, a, frames, n_local):
        out = np.zeros(n_local + 2, np.uint32)
        n = self.lib.orc_build_local_window(a, frames, n_local, _p(out, _u32p))
        if n < 0:
            raise IndexError("query frame outside video")
        return out[:n].tolist()

    def build_global_index_set(self, frames, n_global):
        out = np.zeros(max(n_global, 1), np.uint32)
        n = self.lib.orc_build_global_index_set(frames, n_global, _p(out, _u32p))
        if n < 0:
            raise ValueError("global set size exceeds frame count")
        return out[:n].tolist()

    def attention_full(self, v, wq, wk, wv, wo, scale, want_row_sums=False):
        v = f32(v)
        F, H, W, Cc = v.shape
        out = np.empty_like(v)
        rs = np.empty(F * H * W, np.float64) if want_row_sums else None
        rc = self.lib.orc_attention_full(_p(v, _f32p), F, H, W, Cc, _p(f32(wq), _f32p),
                                         _p(f32(wk), _f32p), _p(f32(wv), _f32p),
                                         _p(f32(wo), _f32p), C.c_float(scale), _p(out, _f32p),
                                         _p(rs, _f64p))
        assert rc == 0, rc
        return (out, rs) if want_row_sums else out

    def dual_scope(self, v, t, wq, wk, wv, wo, scale, n_local=16, n_global=16, bias=10.0,
                   t_star=800.0, heads=1, counters=False):
        v = f32(v)
        F, H, W, Cc = v.shape
        out = np.empty_like(v)
        cnt = np.zeros(3, np.uint64)
        rc = self.lib.orc_dual_scope(_p(v, _f32p), F, H, W, Cc, C.c_double(t), _p(f32(wq), _f32p),
                                     _p(f32(wk), _f32p), _p(f32(wv), _f32p), _p(f32(wo), _f32p),
                                     C.c_float(scale), heads, n_local, n_global, C.c_float(bias),
                                     C.c_double(t_star), _p(out, _f32p), _p(cnt, _u64p))
        if rc:
            raise ValueError(f"dual_scope rc={rc}")
        return (out, cnt.tolist()) if counters else out

    def attention_parallel(self, frames, workers, worker, v, pre, post, glob, t, wq, wk, wv, wo,
                           scale, n_local=16, n_global=16, bias=10.0, t_star=800.0, heads=1):
        v = f32(v)
        Fc, H, W, Cc = v.shape
        out = np.empty_like(v)
        rc = self.lib.orc_attention_parallel(
            frames, workers, worker, _p(v, _f32p), _p(None if pre is None else f32(pre), _f32p),
            _p(None if post is None else f32(post), _f32p),
            _p(None if glob is None else f32(glob), _f32p), H, W, Cc, C.c_double(t),
            _p(f32(wq), _f32p), _p(f32(wk), _f32p), _p(f32(wv), _f32p), _p(f32(wo), _f32p),
            C.c_float(scale), heads, n_local, n_global, C.c_float(bias), C.c_double(t_star),
            _p(out, _f32p))
        if rc:
            raise ValueError(f"attention_parallel rc={rc}")
        return out

    def global_members_in_range(self, frames, n_global, start, length):
        out = np.zeros(max(n_global, 1), np.uint32)
        n = self.lib.orc_global_members_in_range(frames, n_global, start, length, _p(out, _u32p))
        return out[:n].tolist()

    def predict_sync_traffic(self, frames, workers, halo, global_frames, worker, frame_bytes):
        out = np.zeros(3, np.uint64)
        rc = self.lib.orc_predict_sync_traffic(frames, workers, halo, global_frames, worker,
                                               C.c_uint64(frame_bytes), _p(out, _u64p))
        assert rc == 0
        return out.tolist()

    def predict_groupnorm_traffic(self, frames, workers, groups, worker):
        out = np.zeros(3, np.uint64)
        rc = self.lib.orc_predict_groupnorm_traffic(frames, workers, groups, worker, _p(out, _u64p))
        assert rc == 0
        return out.tolist()

    def block_forward(self, x, bp: BlockParams, t, groups, n_local=16, n_global=16, bias=10.0,
                      t_star=800.0, eps=1e-5, heads=1, scale=None):
        x = f32(x)
        F, H, W, Cc = x.shape
        if scale is None:
            scale = float(np.float32(1.0) / np.sqrt(np.float32(Cc)))
        out = np.empty_like(x)
        rc = self.lib.orc_block_forward(
            _p(x, _f32p), F, H, W, Cc, bp.taps, groups, C.c_double(t),
            *[_p(a, _f32p) for a in bp.arrays()[:6]], C.c_float(eps),
            *[_p(a, _f32p) for a in bp.arrays()[6:]], C.c_float(scale), heads, n_local, n_global,
            C.c_float(bias), C.c_double(t_star), _p(out, _f32p))
        if rc:
            raise ValueError(f"block_forward rc={rc}")
        return out


class Reference:
    """The unmodified reference library (oracle/_ref/libvinf_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.lib.ref_last_error.restype = C.c_char_p

    def _chk(self, rc):
        if rc:
            raise RuntimeError(f"reference rc={rc}: {self.lib.ref_last_error().decode()}")

    def fill_seeded(self, n, seed, first_elem=0):
        out = np.empty(n, np.float32)
        self._chk(self.lib.ref_fill_seeded(_p(out, _f32p), C.c_uint64(n), C.c_uint64(seed),
                                           C.c_uint64(first_elem)))
        return out

    def build_block(self, C_, taps=3, groups=1, weight_seed=1, blocks=1, block=0) -> BlockParams:
        bp = BlockParams(C_, taps)
        self._chk(self.lib.ref_build_block(C_, taps, groups, C.c_uint64(weight_seed), blocks,
                                           block, *[_p(a, _f32p) for a in bp.arrays()]))
        return bp

    def conv_over_extended(self, ext, out_start, out_len, taps, w, b):
        ext = f32(ext)
        F, H, W, Cc = ext.shape
        out = np.empty((out_len, H, W, Cc), np.float32)
        self._chk(self.lib.ref_conv_over_extended(_p(ext, _f32p), F, H, W, Cc, out_start, out_len,
                                                  taps, _p(f32(w), _f32p), _p(f32(b), _f32p),
                                                  _p(out, _f32p)))
        return out

    def group_norm(self, v, groups, gamma, beta, eps=1e-5, stats=False):
        v = f32(v)
        F, H, W, Cc = v.shape
        out = np.empty_like(v)
        m = np.empty(groups, np.float64)
        s = np.empty(groups, np.float64)
        self._chk(self.lib.ref_group_norm(_p(v, _f32p), F, H, W, Cc, groups, _p(f32(gamma), _f32p),
                                          _p(f32(beta), _f32p), C.c_float(eps), _p(out, _f32p),
                                          _p(m, _f64p), _p(s, _f64p)))
        return (out, m, s) if stats else out

    def dual_scope(self, v, t, wq, wk, wv, wo, scale, n_local=16, n_global=16, bias=10.0,
                   t_star=800.0, counters=False):
        v = f32(v)
        F, H, W, Cc = v.shape
        out = np.empty_like(v)
        cnt = np.zeros(3, np.uint64)
        self._chk(self.lib.ref_dual_scope(_p(v, _f32p), F, H, W, Cc, C.c_double(t),
                                          _p(f32(wq), _f32p), _p(f32(wk), _f32p),
                                          _p(f32(wv), _f32p), _p(f32(wo), _f32p), C.c_float(scale),
                                          n_local, n_global, C.c_float(bias), C.c_double(t_star),
                                          _p(out, _f32p), _p(cnt, _u64p)))
        return (out, cnt.tolist()) if counters else out

    def attention_full(self, v, wq, wk, wv, wo, scale, want_row_sums=False):
        v = f32(v)
        F, H, W, Cc = v.shape
        out = np.empty_like(v)
        rs = np.empty(F * H * W, np.float64) if want_row_sums else None
        self._chk(self.lib.ref_attention_full(_p(v, _f32p), F, H, W, Cc, _p(f32(wq), _f32p),
                                              _p(f32(wk), _f32p), _p(f32(wv), _f32p),
                                              _p(f32(wo), _f32p), C.c_float(scale),
                                              _p(out, _f32p), _p(rs, _f64p)))
        return (out, rs) if want_row_sums else out

    def build_local_window(self, a, frames, n_local):
        out = np.zeros(n_local + 2, np.uint32)
        n = self.lib.ref_build_local_window(a, frames, n_local, _p(out, _u32p))
        if n < 0:
            raise IndexError(self.lib.ref_last_error().decode())
        return out[:n].tolist()

    def build_global_index_set(self, frames, n_global):
        out = np.zeros(max(n_global, 1), np.uint32)
        n = self.lib.ref_build_global_index_set(frames, n_global, _p(out, _u32p))
        if n < 0:
            raise ValueError(self.lib.ref_last_error().decode())
        return out[:n].tolist()

    def global_members_in_range(self, frames, n_global, start, length):
        out = np.zeros(max(n_global, 1), np.uint32)
        n = self.lib.ref_global_members_in_range(frames, n_global, start, length, _p(out, _u32p))
        return out[:n].tolist()

    def predict_sync_traffic(self, frames, workers, halo, global_frames, worker, frame_bytes):
        out = np.zeros(3, np.uint64)
        self._chk(self.lib.ref_predict_sync_traffic(frames, workers, halo, global_frames, worker,
                                                    C.c_uint64(frame_bytes), _p(out, _u64p)))
        return out.tolist()

    def predict_groupnorm_traffic(self, frames, workers, groups, worker):
        out = np.zeros(3, np.uint64)
        self._chk(self.lib.ref_predict_groupnorm_traffic(frames, workers, groups, worker,
                                                         _p(out, _u64p)))
        return out.tolist()

    def block_forward(self, x, taps, groups, weight_seed, t, n_local=16, n_global=16, bias=10.0,
                      t_star=800.0, workers=0, traffic=False):
        x = f32(x)
        F, H, W, Cc = x.shape
        out = np.empty_like(x)
        bpk = np.zeros(3 * max(workers, 1), np.uint64)
        self._chk(self.lib.ref_block_forward(_p(x, _f32p), F, H, W, Cc, taps, groups,
                                             C.c_uint64(weight_seed), n_local, n_global,
                                             C.c_float(bias), C.c_double(t_star), C.c_double(t),
                                             workers, _p(out, _f32p), _p(bpk, _u64p)))
        return (out, bpk.reshape(-1, 3).tolist()) if traffic else out

    def execute_run(self, F, H, W, Cc, groups=32, n_local=16, n_global=16, blocks=1, steps=1,
                    workers=0, seed=0, weight_seed=1, want_x0=False):
        x0 = np.empty((F, H, W, Cc), np.float32) if want_x0 else None
        wall = C.c_double(0.0)
        self._chk(self.lib.ref_execute_run(F, H, W, Cc, groups, n_local, n_global, blocks, steps,
                                           workers, C.c_uint64(seed), C.c_uint64(weight_seed),
                                           _p(x0, _f32p), C.byref(wall)))
        return (wall.value, x0) if want_x0 else wall.value


class ReferenceRunAPI:
    """The reference's OWN run-level C API (include/vinf.h:27-75) as exported by
    oracle/_ref/libvinf_ref.so (its capi.cpp compiled in) — the checker for
    include/vinf_run.h. Methods return (status, value) so tests can compare codes."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        vp = C.c_void_p
        sigs = {
            "vinf_config_create": (C.c_int, [C.POINTER(vp)]),
            "vinf_config_destroy": (None, [vp]),
            "vinf_config_load_file": (C.c_int, [vp, C.c_char_p]),
            "vinf_config_set": (C.c_int, [vp, C.c_char_p, C.c_char_p]),
            "vinf_config_validate": (C.c_int, [vp]),
            "vinf_config_digest": (C.c_int, [vp, _u64p]),
            "vinf_config_canonical": (C.c_int, [vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
            "vinf_run": (C.c_int, [vp, C.c_char_p, C.c_char_p, _f64p]),
            "vinf_verify": (C.c_int, [C.c_char_p, C.c_char_p, C.c_double, _f64p, _u64p]),
            "vinf_bench": (C.c_int, [vp, _u32p, C.c_size_t, C.c_char_p, C.c_char_p, C.c_size_t,
                                     C.POINTER(C.c_size_t)]),
            "vinf_validate_schedule": (C.c_int, [C.c_uint32, C.c_int, C.POINTER(C.c_int), _u32p,
                                                 _u64p, C.c_char_p, C.c_size_t]),
            "vinf_last_error": (C.c_char_p, []),
        }
        for n, (r, a) in sigs.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        self.lib = L

    def config(self, values: dict | None = None, path: str | None = None):
        h = C.c_void_p()
        assert self.lib.vinf_config_create(C.byref(h)) == 0
        rc = 0
        if path is not None:
            rc = self.lib.vinf_config_load_file(h, path.encode())
        for k, v in (values or {}).items():
            if rc == 0:
                rc = self.lib.vinf_config_set(h, str(k).encode(), str(v).encode())
        return h, rc

    def free(self, h):
        self.lib.vinf_config_destroy(h)

    def canonical(self, h) -> str:
        buf = C.create_string_buffer(8192)
        n = C.c_size_t()
        assert self.lib.vinf_config_canonical(h, buf, 8192, C.byref(n)) == 0
        return buf.value.decode()

    def digest(self, h) -> int:
        d = C.c_uint64()
        assert self.lib.vinf_config_digest(h, C.byref(d)) == 0
        return d.value

    def run(self, h, out_path=None, metrics_path=None):
        wall = C.c_double()
        rc = self.lib.vinf_run(h, out_path.encode() if out_path else None,
                               metrics_path.encode() if metrics_path else None, C.byref(wall))
        return rc, wall.value

    def verify(self, a, b, tol):
        md, bad = C.c_double(), C.c_uint64()
        rc = self.lib.vinf_verify(a.encode(), b.encode(), tol, C.byref(md), C.byref(bad))
        return rc, md.value, bad.value

    def bench(self, h, sweep, metrics_path=None):
        arr = (C.c_uint32 * max(1, len(sweep)))(*sweep)
        buf = C.create_string_buffer(1 << 16)
        n = C.c_size_t()
        rc = self.lib.vinf_bench(h, arr, len(sweep), metrics_path.encode() if metrics_path else None,
                                 buf, 1 << 16, C.byref(n))
        return rc, buf.value.decode()

    def validate_schedule(self, workers, literal):
        done, rounds, transfers = C.c_int(), C.c_uint32(), C.c_uint64()
        buf = C.create_string_buffer(4096)
        rc = self.lib.vinf_validate_schedule(workers, int(literal), C.byref(done), C.byref(rounds),
                                             C.byref(transfers), buf, 4096)
        return rc, bool(done.value), rounds.value, transfers.value, buf.value.decode()
