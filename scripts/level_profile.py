"""Per-kernel breakdown of one engine shape (diagnostic):
    python scripts/level_profile.py F H W C [steps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_16260_b200 import engine as en, ops
F, H, W, C = map(int, sys.argv[1:5])
steps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
d = en.make_desc(F, 1, 0, H, W, C, 3, 32, 1, 16, 16, 10.0, 800.0, 1e-5, 0.0, 1, torch.bfloat16)
e = en.ClipEngine(en.Layout(d))
e.init_weights(1)
e.x.copy_(ops.tensor_from_seed((F, H, W, C), 0, dtype=torch.bfloat16, device="cuda"))
for _ in range(2):
    e.forward_single(900.0)
torch.cuda.synchronize()
e.profile(True)
e.kernel_stats()
for _ in range(steps):
    e.forward_single(900.0)
torch.cuda.synchronize()
st = e.kernel_stats()
tot = sum(v[0] for v in st.values()) / steps
print(f"F={F} {H}x{W} C={C}: {tot:.3f} ms/step")
for k, (ms, n) in st.items():
    print(f"  {k:12s} {ms / steps * 1000:9.1f} us/step  ({n // steps} launches/step)")
