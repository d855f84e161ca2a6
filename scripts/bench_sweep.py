"""BASELINE configs[4]: global-context frame count x local window sweep vs throughput and
roofline fraction, at the configs[1] block shape (40x64 latent, C=640, bf16, 1 GPU).

    python scripts/bench_sweep.py [--steps K] [--out gpurun_out/cfg5_sweep.json]

n_global <= F and n_local / 2 <= F: at the 24-frame clip n_global runs 4..16; the 64-frame
rows extend it to 32 and 64, the 288-frame rows (one GPU's clip of 2,304 frames over 8) run
4..64 at long-clip block shapes. Each point: frames/s of the whole block (device-resident, CUDA
events), the attention core's time and its HBM roofline fraction (Q, K, V read once + ctx
written), and the block's fraction of the sustained tensor peak."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

H, W, C = 40, 64, 640


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "cfg5_sweep.json"))
    args = ap.parse_args()
    import torch

    from bench import peaks
    from paper_2406_16260_b200 import engine as en
    from paper_2406_16260_b200 import ops
    hbm, _, tf_sus, src = peaks()
    points = [(24, g, l) for g in (4, 8, 16) for l in (2, 4, 8, 16, 32)]
    points += [(64, g, l) for g in (32, 64) for l in (2, 8, 16, 32)]
    # one GPU's clip of the 2,304-frame video over 8 GPUs: long clips, where the window band
    # and the sampled globals make 32-query blocks with up to 95 distinct K/V frames
    points += [(288, g, l) for g in (4, 16, 64) for l in (2, 16, 32)]
    rows = []
    for F, ng, nl in points:
        d = en.make_desc(F, 1, 0, H, W, C, 3, 32, 1, nl, ng, 10.0, 800.0, 1e-5, 0.0, 1, torch.bfloat16)
        e = en.ClipEngine(en.Layout(d))
        e.init_weights(1)
        e.x.copy_(ops.tensor_from_seed((F, H, W, C), 0, dtype=torch.bfloat16, device="cuda"))
        for _ in range(args.warmup):
            e.forward_single(900.0)
        torch.cuda.synchronize()
        e.profile(True)
        e.kernel_stats()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            e.forward_single(900.0)
        b.record()
        torch.cuda.synchronize()
        st = e.kernel_stats()
        ms = a.elapsed_time(b) / args.steps
        attn_ms = st["attn_core"][0] / st["attn_core"][1]
        fused = "o_gemm" not in st  # one head: the O projection absorbed into V, output fused
        attn_bytes = (5.0 if fused else 4.0) * F * H * W * C * 2
        flops = (12.0 if fused else 14.0) * F * H * W * C * C
        row = {"frames": F, "n_global": ng, "n_local": nl, "ms_per_step": ms,
               "frames_per_s": F / (ms / 1000.0), "attn_core_us": attn_ms * 1000.0, "fused_output": fused,
               "attn_core_gbs": attn_bytes / (attn_ms / 1000.0) / 1e9,
               "attn_core_frac_hbm": attn_bytes / (attn_ms / 1000.0) / 1e9 / hbm,
               "block_frac_tensor": flops / (ms / 1000.0) / 1e12 / tf_sus}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del e
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump({"workload": "BASELINE configs[4] sweep at configs[1] shape (40x64, C=640, bf16, 1 GPU)",
                   "peaks": {"hbm_gbs": hbm, "tensor_tflops_sustained": tf_sus, "source": src},
                   "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
