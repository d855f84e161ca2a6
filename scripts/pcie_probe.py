"""PCIe probe: pinned H2D alone, D2H alone, and both directions concurrently, for the
bench clip size (78.6 MB bf16), to bound the e2e number."""
import torch

n = 24 * 40 * 64 * 640
h_in = torch.empty(n, dtype=torch.bfloat16, pin_memory=True)
h_out = torch.empty(n, dtype=torch.bfloat16, pin_memory=True)
d_a = torch.empty(n, dtype=torch.bfloat16, device="cuda")
d_b = torch.empty(n, dtype=torch.bfloat16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d():
    d_a.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_b, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


mb = n * 2 / 1e6
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = timed(fn)
    print(f"{name}: {ms:.3f} ms/step  {mb / ms:.1f} GB/s per direction  -> {24 / ms * 1000:.0f} frames/s if PCIe-bound")
