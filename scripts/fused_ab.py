"""Fused Q/K/V+attention kernel vs the unfused path: bitwise equality and step time."""
import json, os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1:
    sys.path.insert(0, ROOT)
    import torch
    from paper_2406_16260_b200 import engine as en, ops
    F, H, W, C = (int(x) for x in sys.argv[2:6])
    d = en.make_desc(F, 1, 0, H, W, C, 3, 32 if C % 32 == 0 else 8, 1, 16, 16, 10.0, 800.0, 1e-5, 0.0, 1,
                     torch.bfloat16)
    e = en.ClipEngine(en.Layout(d)); e.init_weights(1)
    e.x.copy_(ops.tensor_from_seed((F, H, W, C), 0, dtype=torch.bfloat16, device="cuda"))
    for t in (900.0, 700.0):
        e.forward_single(t)
        torch.cuda.synchronize()
        np.save(f"/tmp/fused_{sys.argv[1]}_{int(t)}.npy", e.y.view(torch.int16).cpu().numpy())
    for _ in range(5): e.forward_single(900.0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(50): e.forward_single(900.0)
    b.record(); torch.cuda.synchronize()
    e.profile(True); e.kernel_stats()
    for _ in range(10): e.forward_single(900.0)
    torch.cuda.synchronize()
    st = e.kernel_stats()
    print(json.dumps({"us": a.elapsed_time(b) / 50 * 1000,
                      "kernels": {k: v[0] / max(v[1], 1) * 1000 for k, v in st.items()}}))
    sys.exit(0)
for shape in (["24", "40", "64", "640"], ["24", "4", "8", "64"], ["24", "40", "64", "320"]):
    res = {}
    for tag, env in (("fused", {"VINF_FUSED_ATTN": "1"}), ("unfused", {})):
        r = subprocess.run([sys.executable, __file__, tag, *shape], capture_output=True, text=True,
                           env=dict(os.environ, **env), timeout=600)
        if r.returncode:
            print(tag, shape, r.stderr[-2000:]); sys.exit(1)
        res[tag] = json.loads(r.stdout.strip().splitlines()[-1])
    same = all(np.array_equal(np.load(f"/tmp/fused_fused_{t}.npy"), np.load(f"/tmp/fused_unfused_{t}.npy"))
               for t in (900, 700))
    print(shape, "bitwise_equal", same, "step us fused %.1f unfused %.1f" % (res["fused"]["us"], res["unfused"]["us"]))
    print("   fused  ", {k: round(v, 1) for k, v in res["fused"]["kernels"].items()})
    print("   unfused", {k: round(v, 1) for k, v in res["unfused"]["kernels"].items()})
