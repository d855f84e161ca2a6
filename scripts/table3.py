"""The paper's Table 3 methodology (sync ablation; the reference's
run_bench ablation rows, runner.cpp:292-300) on ONE B200: N clip-parallel workers of the
cfg2/cfg3 block (24 frames per worker, 40x64, C=640, 16 globals, bf16) run as in-process
workers of the C++ executor (comm.local_comms: one host thread per worker, exchanges as
device copies inside one HBM; NVLink is not exercised here). For each N it times the full
block step and the step with each sync kind ablated, and reports the exchanges' own device
time per kind (engine profiling spans on the comm stream).

    python scripts/table3.py [--workers 1 2 4 8] [--steps 10] [--out profiles/r02_table3.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2406_16260_b200 import engine as en  # noqa: E402
from paper_2406_16260_b200 import ops  # noqa: E402
from paper_2406_16260_b200.comm import local_comms  # noqa: E402

F_CLIP, H, W, C = 24, 40, 64, 640


def build(n, ablate):
    F = F_CLIP * n
    engines = []
    for w in range(n):
        d = en.make_desc(F, n, w, H, W, C, 3, 32, 1, 16, 16, 10.0, 800.0, 1e-5, 0.0, 1, torch.bfloat16)
        e = en.ClipEngine(en.Layout(d))
        e.init_weights(1)
        e.set_ablation(ablate)
        e.x.copy_(ops.tensor_from_seed((F_CLIP, H, W, C), 0, first_elem=w * F_CLIP * H * W * C,
                                       dtype=torch.bfloat16, device="cuda"))
        engines.append(e)
    return engines


def time_step(engines, group, steps):
    for _ in range(3):
        en.forward(900.0, engines, group)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        en.forward(900.0, engines, group)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = []
    for n in args.workers:
        rec = {"workers": n, "frames": F_CLIP * n}
        for ablate in (None, "conv", "groupnorm", "attention"):
            engines = build(n, ablate)
            group = en.CommGroup(local_comms(n), use_graph=False) if n > 1 else None
            ms = time_step(engines, group, args.steps)
            rec["ms_" + (ablate or "full")] = ms
            if ablate is None:
                for e in engines:
                    e.profile(True)
                    e.kernel_stats()
                en.forward(900.0, engines, group)
                torch.cuda.synchronize()
                kinds = {}
                for e in engines:
                    for k, (t, _) in e.kernel_stats().items():
                        kinds[k] = kinds.get(k, 0.0) + t
                    e.profile(False)
                rec["spans_ms_all_workers"] = kinds
                rec["sync_ms_per_worker"] = {k: kinds.get(k, 0.0) / n for k in ("xchg_conv", "allreduce_gn", "xchg_attn")}
                rec["bytes_sent_per_worker"] = (
                    [sum(x.bytes for st in (0, 1) for x in e.layout.exchange(st) if x.send) for e in engines])
            del engines
            torch.cuda.empty_cache()
        full = rec["ms_full"]
        rec["overhead_vs_ablated_pct"] = {k: 100.0 * (full - rec["ms_" + k]) / full for k in
                                          ("conv", "groupnorm", "attention")}
        rows.append(rec)
        print(json.dumps(rec), flush=True)
    out = {"what": "sync ablation on one B200 (in-process workers of the C++ executor; exchanges are device "
                   "copies in one HBM, NVLink not exercised); all N workers share the GPU, so ms are the "
                   "whole job's", "config": {"frames_per_worker": F_CLIP, "height": H, "width": W, "channels": C,
                                            "n_local": 16, "n_global": 16, "dtype": "bf16", "t": 900.0},
           "rows": rows}
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
