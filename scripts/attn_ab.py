"""A/B of the two bf16 attention-core kernels (VINF_ATTN_VARIANT=1 ring, 0 pipeline):
bitwise equality of the engine output and per-kernel time, at cfg2 (N=1) and at a
clip-parallel worker with halos + remote globals (R up to 56)."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")


def child(variant: str, workers: int, worker: int):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2406_16260_b200 import engine as en
    from paper_2406_16260_b200 import ops
    F = 24 * workers
    d = en.make_desc(F, workers=workers, worker=worker, height=40, width=64, channels=640, groups=32,
                     n_local=16, n_global=16, dtype=torch.bfloat16)
    engines = []
    for w in range(workers):
        dw = en.make_desc(F, workers=workers, worker=w, height=40, width=64, channels=640, groups=32,
                          n_local=16, n_global=16, dtype=torch.bfloat16)
        ew = en.ClipEngine(en.Layout(dw))
        ew.init_weights(1)
        ew.x.copy_(ops.tensor_from_seed((24, 40, 64, 640), w + 7).to(torch.bfloat16).cuda())
        engines.append(ew)
    e = engines[worker]
    e.profile(True)
    grp = en.LocalGroup() if workers > 1 else None
    for _ in range(3):
        en.forward(900.0, engines, grp)
    torch.cuda.synchronize()
    e.kernel_stats()
    for _ in range(20):
        en.forward(900.0, engines, grp)
    torch.cuda.synchronize()
    st = e.kernel_stats()
    y = e.y.float().cpu().numpy()
    np.save(os.path.join("/tmp", f"attn_ab_{variant}_{workers}.npy"), y)
    print(json.dumps({k: v[0] / max(v[1], 1) * 1000 for k, v in st.items()}))


if __name__ == "__main__":
    if len(sys.argv) > 1:
        child(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]))
        sys.exit(0)
    os.makedirs(OUT, exist_ok=True)
    variants = [("ring", {"VINF_ATTN_VARIANT": "1"})] + [
        (f"lean{n}", {"VINF_ATTN_VARIANT": "0", "VINF_ATTN_STAGES": str(n)}) for n in (4, 5, 6)]
    for workers, worker in ((1, 0), (4, 1)):
        res = {}
        for v, extra in variants:
            env = dict(os.environ, **extra)
            r = subprocess.run([sys.executable, __file__, v, str(workers), str(worker)], env=env,
                               capture_output=True, text=True, timeout=600)
            if r.returncode != 0:
                print(r.stderr[-3000:])
                sys.exit(1)
            res[v] = json.loads(r.stdout.strip().splitlines()[-1])
        a = np.load(os.path.join("/tmp", f"attn_ab_ring_{workers}.npy"))
        for v, _ in variants[1:]:
            b = np.load(os.path.join("/tmp", f"attn_ab_{v}_{workers}.npy"))
            print(f"workers={workers} {v} bitwise_equal={np.array_equal(a.view(np.uint32), b.view(np.uint32))}")
        for k in res["ring"]:
            print(f"  {k:12s} " + "  ".join(f"{v} {res[v].get(k, 0):7.1f}" for v, _ in variants))
