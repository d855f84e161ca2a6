"""HBM write / read / copy bandwidth with plain torch ops (diagnostic): how fast can a kernel
that mostly writes (the Q/K/V projection: 3 bytes out per byte in) move its output?"""
import torch
n = 4 << 30  # bytes
a = torch.empty(n // 2, dtype=torch.bfloat16, device="cuda")
b = torch.empty_like(a)
a.fill_(1.0)
def t(f, reps=10):
    f(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(reps):
        s.record(); f(); e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e))
    return best
w = t(lambda: b.fill_(2.0))
r = t(lambda: a.sum(dtype=torch.float32))
c = t(lambda: b.copy_(a))
print(f"write {n / w / 1e6:.0f} GB/s  read {n / r / 1e6:.0f} GB/s  copy (r+w) {2 * n / c / 1e6:.0f} GB/s")
