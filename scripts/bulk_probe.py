"""TMA bulk-copy feed bandwidth (diagnostics): chunk size x ring depth x CTAs per SM."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_16260_b200 import _lib
lib = _lib.load(); ms = C.c_float()
B = 2 << 30
_lib.check(lib.vinf_read_bw_bench(B, 10, C.byref(ms))); print(f"LDG stream: {B / ms.value / 1e6:.0f} GB/s")
for chunk in (4096, 8192, 16384):
    for stages, ctas in ((4, 4), (7, 3), (12, 2), (24, 1)):
        if stages * chunk * ctas > 220 * 1024: continue
        _lib.check(lib.vinf_bulk_bw_bench(B, chunk, stages, ctas, 10, C.byref(ms)))
        print(f"bulk chunk {chunk:6d} stages {stages:2d} ctas {ctas}: {B / ms.value / 1e6:6.0f} GB/s  ({stages*chunk*ctas//1024} KB in flight/SM)")
