"""Small engine runs for compute-sanitizer (memcheck / synccheck / racecheck): every kernel
family of the product path (stub, conv GEMM + GroupNorm statistics, fold / apply, Q/K/V and
O GEMMs with TMA epilogues, the attention core, Euler) in both arithmetic modes, one worker
and two in-process workers over the C++ executor.
    compute-sanitizer --tool memcheck python scripts/sanitize_case.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2406_16260_b200 import engine as en  # noqa: E402
from paper_2406_16260_b200 import ops  # noqa: E402
from paper_2406_16260_b200.comm import local_comms  # noqa: E402


def run(F, H, W, C, n, dtype, heads=1, n_local=8, n_global=8):
    x = ops.tensor_from_seed((F, H, W, C), 0, dtype=dtype, device="cuda")
    engines = []
    for w in range(n):
        d = en.make_desc(F, n, w, H, W, C, 3, 8, heads, n_local, n_global, 10.0, 800.0, 1e-5, 0.0, 1, dtype)
        e = en.ClipEngine(en.Layout(d))
        e.init_weights(1)
        e.x.copy_(x[e.layout.start:e.layout.start + e.layout.f_clip])
        engines.append(e)
    group = en.CommGroup(local_comms(n), use_graph=False) if n > 1 else None
    en.forward(900.0, engines, group)
    en.forward(700.0, engines, group)
    torch.cuda.synchronize()
    y = torch.cat([e.y.float() for e in engines])
    assert torch.isfinite(y).all()
    print(f"ok F={F} {H}x{W} C={C} workers={n} {dtype} heads={heads}", flush=True)


if __name__ == "__main__":
    run(24, 2, 16, 64, 1, torch.bfloat16)
    run(24, 2, 16, 64, 1, torch.float32)
    run(24, 2, 16, 128, 2, torch.bfloat16, heads=2)
    run(48, 1, 32, 64, 2, torch.float32, n_global=16)
