"""Per-kernel breakdown of one clip-parallel worker's block step (diagnostic): the engine of
worker w of N at the bench shape, its stages run in order with the exchanges skipped, so the
kernels are exactly those of a real N-GPU step (the halo / remote-global slots are left as
they are): python scripts/worker_profile.py N [w] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2406_16260_b200 import _lib, engine as en, ops

N = int(sys.argv[1])
w = int(sys.argv[2]) if len(sys.argv) > 2 else N // 2
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
F, H, W, C = 24 * N, 40, 64, 640
d = en.make_desc(F, N, w, H, W, C, 3, 32, 1, 16, 16, 10.0, 800.0, 1e-5, 0.0, 1, torch.bfloat16)
e = en.ClipEngine(en.Layout(d))
e.init_weights(1)
e.x.copy_(ops.tensor_from_seed((24, H, W, C), 0, dtype=torch.bfloat16, device="cuda"))


def step():
    for st in (_lib.VINF_STAGE_STUB, _lib.VINF_STAGE_CONV, _lib.VINF_STAGE_GN_APPLY, _lib.VINF_STAGE_QKV,
               _lib.VINF_STAGE_ATTENTION):
        e.stage(0, st, 900.0)


for _ in range(3):
    step()
torch.cuda.synchronize()
s0, s1 = torch.cuda.Event(True), torch.cuda.Event(True)
s0.record()
for _ in range(steps):
    step()
s1.record()
torch.cuda.synchronize()
ms = s0.elapsed_time(s1) / steps
e.profile(True)
e.kernel_stats()
for _ in range(steps):
    step()
torch.cuda.synchronize()
st = e.kernel_stats()
print(f"worker {w} of {N} (24 frames/GPU, 40x64, C=640, bf16): {ms * 1000:.1f} us/step "
      f"({24 / ms * 1000:.0f} frames/s/GPU), exchanges skipped")
for k, (t, n) in st.items():
    print(f"  {k:12s} {t / steps * 1000:9.1f} us/step  ({n // steps} launches/step)")
