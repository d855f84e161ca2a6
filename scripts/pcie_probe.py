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

# the same bidirectional transfer split into k chunks on k streams per direction
for k in (2, 4):
    ups = [torch.cuda.Stream() for _ in range(k)]
    downs = [torch.cuda.Stream() for _ in range(k)]
    c = n // k

    def both_k():
        cur = torch.cuda.current_stream()
        for i in range(k):
            ups[i].wait_stream(cur)
            downs[i].wait_stream(cur)
            with torch.cuda.stream(ups[i]):
                d_a[i * c:(i + 1) * c].copy_(h_in[i * c:(i + 1) * c], non_blocking=True)
            with torch.cuda.stream(downs[i]):
                h_out[i * c:(i + 1) * c].copy_(d_b[i * c:(i + 1) * c], non_blocking=True)
        for i in range(k):
            cur.wait_stream(ups[i])
            cur.wait_stream(downs[i])

    ms = timed(both_k)
    print(f"both x{k} streams: {ms:.3f} ms/step  {mb / ms:.1f} GB/s per direction  -> {24 / ms * 1000:.0f} frames/s")
