"""Diagnostic: sha256 of the bf16 engine output at an engine shape (compare across builds or
environment switches for bitwise equality): python scripts/diag_hash.py [F H W C]"""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_16260_b200 import engine as en, ops
F, H, W, C = map(int, sys.argv[1:5]) if len(sys.argv) > 4 else (24, 40, 64, 640)
desc = en.make_desc(F, 1, 0, H, W, C, 3, 32, 1, 16, 16, 10.0, 800.0, 1e-5, 0.0, 1, torch.bfloat16)
e = en.ClipEngine(en.Layout(desc)); e.init_weights(1)
e.x.copy_(ops.tensor_from_seed((F, H, W, C), 0, dtype=torch.bfloat16, device="cuda"))
for t in (900.0, 700.0):
    en.forward(t, [e]); torch.cuda.synchronize()
    print(f"F={F} {H}x{W} C={C} t={t}: {hashlib.sha256(e.y.cpu().view(torch.int16).numpy().tobytes()).hexdigest()[:16]}")
