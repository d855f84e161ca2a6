"""Step time of the cfg2 block: profiled (per-kernel events, no graph) vs graph replay."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_16260_b200 import engine as en, ops
d = en.make_desc(24, 1, 0, 40, 64, 640, 3, 32, 1, 16, 16, 10.0, 800.0, 1e-5, 0.0, 1, torch.bfloat16)
e = en.ClipEngine(en.Layout(d)); e.init_weights(1)
e.x.copy_(ops.tensor_from_seed((24, 40, 64, 640), 0, dtype=torch.bfloat16, device="cuda"))
for prof in (True, False, True, False):
    e.profile(prof)
    for _ in range(5): e.forward_single(900.0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(100): e.forward_single(900.0)
    b.record(); torch.cuda.synchronize()
    if prof: e.kernel_stats()
    print("profiled" if prof else "graph   ", round(a.elapsed_time(b) / 100 * 1000, 1), "us/step")
