"""B200-native (sm_100a) clip-parallel dual-scope temporal block (Video-Infinity,
arXiv 2406.16260): hand-written CUDA kernels behind a C ABI (include/vinf_temporal.h),
with a Python host layer mirroring the reference temporal-module API."""
from . import _lib  # noqa: F401

__all__ = ["ops", "clip_parallel", "engine", "transport"]
