"""GEMM microbenchmark (diagnostic): main loop vs epilogue cost at the bench shapes.
    python scripts/gemm_micro.py [shape ...]   (conv, qkv, o, sq8k; default all)"""
import ctypes as C, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_16260_b200 import _lib
L = _lib.load()
M = 24 * 40 * 64
SHAPES = {"conv": (640, 640, 3, 1), "qkv": (1920, 640, 1, 0), "o": (640, 640, 1, 1), "sq8k": (8192, 8192, 1, 0)}
# custom shapes: name=M,N,K,nseg,res (e.g. conv320=5898240,320,320,3,1)
for a in sys.argv[1:]:
    if "=" in a and not a.startswith("--"):
        nm, v = a.split("=")
        m_, n_, k_, s_, r_ = map(int, v.split(","))
        SHAPES[nm] = (n_, k_, s_, r_, m_)
names = [a.split("=")[0] for a in sys.argv[1:] if a.split("=")[0] in SHAPES] or list(SHAPES)
iters = 3 if "--once" in sys.argv else 20
for name in names:
    N, K, nseg, res = SHAPES[name][:4]
    m = SHAPES[name][4] if len(SHAPES[name]) > 4 else (M if name != "sq8k" else 8192)
    fl = [a for a in sys.argv[1:] if a.startswith("--flags=")]
    for flags in ([int(v) for v in fl[0][8:].split(",")] if fl else (0,) if "--once" in sys.argv else (0, 1)):
        ms = C.c_float()
        _lib.check(L.vinf_gemm_bench(m, N, K, nseg, flags, res, iters, C.byref(ms)))
        tf = 2.0 * m * N * K * nseg / (ms.value * 1e-3) / 1e12
        print(f"{name:5s} M={m} N={N} K={K}x{nseg} res={res} flags={flags}: {ms.value*1000:8.1f} us  {tf:7.1f} TFLOP/s")
