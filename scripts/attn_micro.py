"""Attention-core micro-benchmark (diagnostics): the core alone on a single-worker layout's
token table, frame-major vs position-major Q/K/V views, plus a streaming-read probe.
    python scripts/attn_micro.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_16260_b200 import _lib  # noqa: E402

lib = _lib.load()
ms = C.c_float()
if len(sys.argv) > 1:  # one case: F H W C heads n_local n_global f32
    F, H, W, Ch, heads, nl, ng, f32 = map(int, sys.argv[1:9])
    pm = int(sys.argv[9]) if len(sys.argv) > 9 else 0
    _lib.check(lib.vinf_attention_bench(F, H, W, Ch, heads, nl, ng, f32, pm, 3, C.byref(ms)))
    print(f"{sys.argv[1:9]}: {ms.value * 1e3:.1f} us")
    sys.exit(0)
for gb in (1, 4):
    _lib.check(lib.vinf_read_bw_bench(gb << 30, 20, C.byref(ms)))
    print(f"read stream {gb} GiB: {ms.value * 1e3:8.1f} us  {(gb << 30) / ms.value / 1e6:8.1f} GB/s")
cases = [(24, 40, 64, 640, 1, 16, 16), (288, 40, 64, 320, 1, 16, 16),
         (96, 20, 32, 640, 1, 16, 16), (288, 10, 16, 1280, 1, 16, 16)]
for (F, H, W, Ch, heads, nl, ng) in cases:
    for f32 in (0, 1):
        row = []
        for pm in (0,):
            _lib.check(lib.vinf_attention_bench(F, H, W, Ch, heads, nl, ng, f32, pm, 20, C.byref(ms)))
            row.append(ms.value * 1e3)
        qkv = F * H * W * Ch * 3 * 2 * (2 if f32 else 1)
        ctx = F * H * W * Ch * 2 * (2 if f32 else 1)
        print(f"F={F:4d} {H}x{W} C={Ch:4d} heads={heads} {'f32' if f32 else 'bf16'}: frame-major {row[0]:7.1f} us "
              f"({(qkv + ctx) / row[0] / 1e3:6.0f} GB/s)  chunked {row[1]:7.1f} us ({(qkv + ctx) / row[1] / 1e3:6.0f} GB/s)")
