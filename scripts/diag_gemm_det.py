"""Diagnostic: GEMM determinism across repeated runs for several shapes/tiles."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_16260_b200 import _lib
L = _lib.load()
for (M, N, K, nseg, res) in [(61440, 1920, 640, 1, 0), (61440, 640, 640, 1, 1), (61440, 640, 640, 3, 1),
                             (61440, 1280, 640, 1, 0), (61440, 1536, 640, 1, 0), (61440, 1024, 640, 1, 0),
                             (8192, 1920, 640, 1, 0), (61440, 1920, 128, 1, 0)]:
    v = C.c_float()
    _lib.check(L.vinf_gemm_bench(M, N, K, nseg, 2, res, 3, C.byref(v)))
    print(f"M={M} N={N} K={K}x{nseg} res={res}: mismatching elements over 5 reruns = {int(-v.value)}")
