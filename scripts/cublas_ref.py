"""cuBLAS (torch.matmul) timings at the block's GEMM shapes, for context (diagnostic)."""
import torch
M = 61440
shapes = {"conv(K=1920)": (M, 640, 1920), "qkv": (M, 1920, 640), "o": (M, 640, 640)}
for name, (m, n, k) in shapes.items():
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16)
    r = torch.randn(m, n, device="cuda", dtype=torch.bfloat16)
    for label, fn in (("mm", lambda: a @ b.t()), ("addmm(+res)", lambda: torch.addmm(r, a, b.t()))):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20): fn()
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1000
        print(f"{name:14s} {label:12s} {us:7.1f} us  {2*m*n*k/us/1e6:7.1f} TFLOP/s")
