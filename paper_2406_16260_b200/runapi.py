"""Run-level API (include/vinf_run.h): the reference's outer C API (include/vinf.h:27-75)
backed by the device engine. Mirrors the reference's names and error behaviour:

    cfg = RunConfig({"frames": 16, "height": 4, "width": 4, "channels": 8, "workers": 2})
    wall = run(cfg, out_path="x0.vinf", metrics_path="m.txt")
    verify("x0.vinf", "ref.vinf", 1e-4)      # -> (max_diff, mismatches); raises on mismatch
    print(bench(cfg, [1, 2]))                  # sequential + sweep + sync-ablation table
    validate_schedule(4)                       # -> (completed, rounds, transfers, cycle)
"""
from __future__ import annotations

import ctypes as C

from . import _lib


class RunConfig:
    def __init__(self, values: dict | None = None, path: str | None = None):
        self._lib = _lib.load()
        h = C.c_void_p()
        _lib.check(self._lib.vinf_config_create(C.byref(h)))
        self._h = h
        if path is not None:
            _lib.check(self._lib.vinf_config_load_file(h, path.encode()))
        for k, v in (values or {}).items():
            self.set(k, v)

    def set(self, key: str, value) -> None:
        if isinstance(value, bool):
            value = "true" if value else "false"
        _lib.check(self._lib.vinf_config_set(self._h, str(key).encode(), str(value).encode()))

    def validate(self) -> None:
        _lib.check(self._lib.vinf_config_validate(self._h))

    def digest(self) -> int:
        d = C.c_uint64()
        _lib.check(self._lib.vinf_config_digest(self._h, C.byref(d)))
        return d.value

    def canonical(self) -> str:
        n = C.c_size_t()
        _lib.check(self._lib.vinf_config_canonical(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _lib.check(self._lib.vinf_config_canonical(self._h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None and _lib._lib is not None:
            _lib._lib.vinf_config_destroy(self._h)
            self._h = None


def run(cfg: RunConfig, out_path: str | None = None, metrics_path: str | None = None) -> float:
    wall = C.c_double()
    _lib.check(_lib.load().vinf_run(cfg._h, out_path.encode() if out_path else None,
                                    metrics_path.encode() if metrics_path else None,
                                    C.byref(wall)))
    return wall.value


def verify(dump_a: str, dump_b: str, tolerance: float) -> tuple[float, int]:
    md, bad = C.c_double(), C.c_uint64()
    _lib.check(_lib.load().vinf_verify(dump_a.encode(), dump_b.encode(), tolerance, C.byref(md),
                                       C.byref(bad)))
    return md.value, bad.value


def verify_nothrow(dump_a: str, dump_b: str, tolerance: float) -> tuple[int, float, int]:
    md, bad = C.c_double(), C.c_uint64()
    rc = _lib.load().vinf_verify(dump_a.encode(), dump_b.encode(), tolerance, C.byref(md),
                                 C.byref(bad))
    return rc, md.value, bad.value


def bench(cfg: RunConfig, sweep: list[int], metrics_path: str | None = None) -> str:
    arr = (C.c_uint32 * max(1, len(sweep)))(*sweep)
    n = C.c_size_t()
    cap = 1 << 16
    buf = C.create_string_buffer(cap)
    _lib.check(_lib.load().vinf_bench(cfg._h, arr, len(sweep),
                                      metrics_path.encode() if metrics_path else None, buf, cap,
                                      C.byref(n)))
    return buf.value.decode()


def validate_schedule(workers: int, literal_order: bool = False) -> tuple[bool, int, int, str]:
    done, rounds, transfers = C.c_int(), C.c_uint32(), C.c_uint64()
    buf = C.create_string_buffer(4096)
    _lib.check(_lib.load().vinf_validate_schedule(workers, int(literal_order), C.byref(done),
                                                  C.byref(rounds), C.byref(transfers), buf, 4096))
    return bool(done.value), rounds.value, transfers.value, buf.value.decode()
