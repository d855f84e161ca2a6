"""e2e pipeline timeline (diagnostic): the bench's two-engine H2D / compute / D2H loop with a
timing event at the start and end of every transfer and step; prints mean durations and gaps.
    python scripts/e2e_timeline.py [steps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_16260_b200 import engine as en, ops

K = int(sys.argv[1]) if len(sys.argv) > 1 else 100
LEAN = "--lean" in sys.argv  # first upload alone waits on the start event
TWO = "--two" in sys.argv  # alternate two upload and two download streams (one per engine)
F, H, W, C = 24, 40, 64, 640
d = en.make_desc(F, 1, 0, H, W, C, 3, 32, 1, 16, 16, 10.0, 800.0, 1e-5, 0.0, 1, torch.bfloat16)
engs = []
for _ in range(2):
    e = en.ClipEngine(en.Layout(d))
    e.init_weights(1)
    engs.append(e)
x = ops.tensor_from_seed((F, H, W, C), 0, dtype=torch.bfloat16, device="cuda")
h_in = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
h_in.copy_(x.cpu())
h_out = [torch.empty_like(h_in, pin_memory=True) for _ in range(2)]
stream = torch.cuda.current_stream()
s_ups = [torch.cuda.Stream(), torch.cuda.Stream()]
s_downs = [torch.cuda.Stream(), torch.cuda.Stream()]
T = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def run(n):
    ev = {k: {} for k in ("u0", "u1", "c0", "c1", "d0", "d1")}
    start = T()
    start.record(stream)

    def upload(j):
        e = engs[j % 2]
        s_up = s_ups[j % 2 if TWO else 0]
        if j == 0 or not LEAN:
            s_up.wait_event(start)
        if j - 2 in ev["c1"]:
            s_up.wait_event(ev["c1"][j - 2])
        ev["u0"][j] = T(); ev["u0"][j].record(s_up)
        with torch.cuda.stream(s_up):
            e.x.copy_(h_in, non_blocking=True)
        ev["u1"][j] = T(); ev["u1"][j].record(s_up)

    upload(0)
    for j in range(n):
        if j + 1 < n:
            upload(j + 1)
        e = engs[j % 2]
        stream.wait_event(ev["u1"][j])
        if j - 2 in ev["d1"]:
            stream.wait_event(ev["d1"][j - 2])
        ev["c0"][j] = T(); ev["c0"][j].record(stream)
        en.forward(900.0, [e])
        ev["c1"][j] = T(); ev["c1"][j].record(stream)
        s_down = s_downs[j % 2 if TWO else 0]
        s_down.wait_event(ev["c1"][j])
        ev["d0"][j] = T(); ev["d0"][j].record(s_down)
        with torch.cuda.stream(s_down):
            h_out[j % 2].copy_(e.y, non_blocking=True)
        ev["d1"][j] = T(); ev["d1"][j].record(s_down)
    end = T()
    stream.wait_event(ev["d1"][n - 1])
    end.record(stream)
    torch.cuda.synchronize()
    return start, end, ev


run(4)
start, end, ev = run(K)
tot = start.elapsed_time(end)
t = lambda k, j: start.elapsed_time(ev[k][j])  # noqa: E731
mean = lambda xs: sum(xs) / len(xs)  # noqa: E731
js = range(2, K - 2)
print(f"lean={LEAN} two={TWO} K={K}: total {tot:.2f} ms, {tot / K:.3f} ms/step, {24 * K / tot * 1000:.0f} frames/s")
print(f"  upload   {mean([t('u1', j) - t('u0', j) for j in js]):.3f} ms, gap before {mean([t('u0', j) - t('u1', j - 1) for j in js]):.3f}")
print(f"  compute  {mean([t('c1', j) - t('c0', j) for j in js]):.3f} ms, gap before {mean([t('c0', j) - t('c1', j - 1) for j in js]):.3f}")
print(f"  download {mean([t('d1', j) - t('d0', j) for j in js]):.3f} ms, gap before {mean([t('d0', j) - t('d1', j - 1) for j in js]):.3f}")
print(f"  first upload ends {t('u1', 0):.3f} ms; last download {t('d0', K - 1):.3f} -> {t('d1', K - 1):.3f} ms")
