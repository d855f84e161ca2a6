"""Isolates the whole-row attention kernel per (C, HW) in fresh processes (diagnostic)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1:
    sys.path.insert(0, ROOT)
    import numpy as np, torch
    from oracle.oracle import Oracle
    from paper_2406_16260_b200 import ops
    orc = Oracle()
    C, H, W = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    x = orc.tensor_from_seed((24, H, W, C), 80)
    bp = orc.build_block(C, weight_seed=81)
    dev = lambda a, dt=torch.float32: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)
    p = ops.AttentionParams(C, dev(bp.wq), dev(bp.wk), dev(bp.wv), dev(bp.wo), heads=1)
    cfg = ops.DualScopeConfig(16, 16, 10.0, 800.0)
    got = ops.dual_scope_reference(dev(x, torch.bfloat16), 900.0, p, cfg)
    torch.cuda.synchronize()
    print("ok", float(got.float().abs().sum()))
    sys.exit(0)
for v, extra in (("1", {}), ("0", {})):
    for C, H, W in ((64, 2, 2), (640, 2, 2), (320, 40, 64)):
        r = subprocess.run([sys.executable, __file__, str(C), str(H), str(W)], capture_output=True, text=True,
                           env=dict(os.environ, VINF_ATTN_VARIANT=v, **extra), timeout=300)
        print(v, C, H, W, r.stdout.strip()[-30:].replace(chr(10), ' '), [l for l in r.stderr.splitlines() if "bulk attn" in l][:1], r.stderr.strip().splitlines()[-1][-100:] if r.returncode else "")
