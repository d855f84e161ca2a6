"""Benchmark: temporal-layer latent frames/s of the clip-parallel dual-scope temporal block
(BASELINE.json metric) on 1..8 B200s, with roofline and CPU-reference context.

    python bench.py [--gpus N --steps K --warmup W --dtype bf16|f32]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU, NCCL)
    python bench.py --impl reference ...                      (reference CPU arm)

A step = one pass of the temporal block (stub -> temporal conv + residual -> GroupNorm
-> dual-scope attention + residual, pipeline.cpp:150-170) over this GPU's clip of
BASELINE configs[1]/[2]: 24 frames per GPU of a 40x64 latent, C=640, 16 global frames
(n_local 16, bias 10, groups 32, taps 3, heads 1 = the reference's single-head form).
Weak scaling: F = 24 * N frames over N GPUs with the 3-step context sync every step.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "temporal-layer latent frames/s at 1/2/4/8 B200; % of HBM/tensor roofline"
FRAMES_PER_GPU, H, W, C = 24, 40, 64, 640
N_LOCAL, N_GLOBAL, GROUPS, TAPS, HEADS, BIAS, T_STAR = 16, 16, 32, 3, 1, 10.0, 800.0
T_STEP = 900.0  # t > t_star: bias on the global tokens (first denoising steps)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-hw", type=int, default=8, help="spatial crop side for CPU arms")
    ap.add_argument("--workload", default="cfg2", choices=["cfg2", "vc2"],
                    help="cfg2: BASELINE configs[1]/[2] (default, the headline); vc2: configs[3], "
                         "the VideoCrafter2-shaped level stack over --frames frames (strong scaling)")
    ap.add_argument("--frames", type=int, default=2300,
                    help="vc2 workload: total frames (uneven clips when the GPU count does not divide it)")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the torch.distributed/NCCL exchange path even with one rank")
    ap.add_argument("--no-f32", action="store_true", help="skip the fp32-mode record")
    ap.add_argument("--no-vc2", action="store_true", help="skip the configs[3] 2,300-frame stack record")
    ap.add_argument("--executor", default="native", choices=["native", "python"],
                    help="N>1: native = the C++ executor (vinf_engine_forward_dist over an NCCL "
                         "communicator, CUDA-graph replay); python = the torch.distributed stage loop")
    return ap.parse_args()


# ---- rank launcher --------------------------------------------------------------


def plan_launch(gpus: int, visible: int, environ: dict, script: str, argv: list, port: int):
    """How this invocation runs: None = in this process (WORLD_SIZE set by torchrun, or one
    GPU), else the argv that re-executes it as `gpus` ranks under torch.distributed.run (one
    process per GPU, rendezvous on 127.0.0.1). Raises SystemExit when fewer GPUs than
    requested are visible, so `--gpus N` never silently measures fewer GPUs."""
    world = int(environ.get("WORLD_SIZE", "0") or 0)
    if world:
        if world != gpus:
            raise SystemExit(f"bench.py: --gpus {gpus} but WORLD_SIZE={world}")
        return None
    if gpus < 1:
        raise SystemExit("bench.py: --gpus must be >= 1")
    if visible < gpus:
        raise SystemExit(f"bench.py: --gpus {gpus} requested but only {visible} CUDA device(s) visible")
    if gpus == 1:
        return None
    return ["-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", script, *argv]


def _free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def max_over_ranks(value: float, device=None) -> float:
    """The max of a per-rank time over all ranks (the bench's multi-GPU clock rule)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def kernel_floor_us(frames: int, h: int, w: int, c: int, es: int, hbm_gbs: float, tf: float,
                    fused_o: bool = False) -> dict:
    """Roofline floor of one block step, kernel by kernel (bf16 GroupNorm-folded pipeline):
    each kernel takes at least max(its tensor work / peak, its algorithmic HBM bytes / peak),
    with T = frames*H*W*C*s the bytes of one clip-sized tensor:
      stub  reads + writes the clip                    2 T              (HBM)
      conv  2*H*W*3C^2 flop per frame; A, residual, out 3 T
      QKV   2*H*W*3C^2 flop per frame; in, Q/K/V out   4 T
      attn  Q/K/V in, ctx out                          4 T              (HBM)
      O     2*H*W*C^2 flop per frame; ctx, residual, out 3 T
    GroupNorm statistics and folding are not counted (latency-bound, a few us per step).
    fused_o (one head): no O GEMM; the attention core reads Q/K/V and the residual and writes
    the block output (5 T); W_vo = W_o W_v is 2 C^3 flop."""
    t = frames * h * w * c * es
    m = frames * h * w
    parts = {"stub": (0.0, 2 * t), "conv_gemm": (6.0 * m * c * c, 3 * t),
             "qkv_gemm": (6.0 * m * c * c, 4 * t), "attn_core": (0.0, 4 * t),
             "o_gemm": (2.0 * m * c * c, 3 * t)}
    if fused_o:
        del parts["o_gemm"]
        parts["attn_core"] = (0.0, 5 * t)
        parts["wvo_gemm"] = (2.0 * c * c * c, 0.0)
    out = {}
    for k, (fl, by) in parts.items():
        out[k] = max(fl / (tf * 1e12), by / (hbm_gbs * 1e9)) * 1e6
    return out


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p["bf16_tflops_sustained"], "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, 1590.0, 1400.0, "fallback"


def tensor_peak(clocks: dict):
    """The bf16 tensor peak that applies to kernels timed under these clocks: the burst
    figure when the SM clock held (median >= 95% of max) with no power cap, else the
    sustained one. Returns (TFLOP/s, which, both)."""
    _, burst, sus, src = peaks()
    mhz, mx = clocks.get("sm_mhz"), clocks.get("sm_max_mhz")
    held = bool(mhz and mx and mhz >= 0.95 * mx and "sw_power_cap" not in clocks.get("reasons", []))
    which = "burst" if held else "sustained"
    return (burst if held else sus), which, {"burst": burst, "sustained": sus, "source": src}


# ---- reference CPU arm ------------------------------------------------------------


def cpu_reference_sample(frames: int, side: int, workers: int, fixed_s: float = 0.0):
    """The reference's own public run path (execute_run, runner.cpp:213-227) on a
    bounded spatial crop (side x side of the 40x64 latent); positions are independent in
    the temporal layers, so frames/s scales by crop/full positions. The run's fixed cost
    (model build, thread start: a side = 1 run, `fixed_s`) is subtracted before scaling, so
    the small crop does not understate the reference. Returns (frames/s at the full 40x64
    size, wall seconds)."""
    from oracle.oracle import Reference
    ref = Reference()
    wall = ref.execute_run(frames, side, side, C, groups=GROUPS, n_local=N_LOCAL, n_global=N_GLOBAL,
                           blocks=1, steps=1, workers=workers)
    work = max(wall - fixed_s, 1e-6)
    return frames / work * (side * side) / (H * W), wall


def cpu_fixed_cost(frames: int, workers: int) -> float:
    """Wall seconds of the reference run at a 1x1 crop: its per-call fixed cost."""
    from oracle.oracle import Reference
    ref = Reference()
    ws = [ref.execute_run(frames, 1, 1, C, groups=GROUPS, n_local=N_LOCAL, n_global=N_GLOBAL, blocks=1,
                          steps=1, workers=workers) for _ in range(3)]
    return sorted(ws)[1]


def ref_workers(frames: int) -> int:
    """The reference's most parallel form on this host: in-process clip-parallel workers
    (it has no intra-op threading), N <= host cores, N | F, and F / N >= the attention halo
    (pipeline.cpp:131-143). 0 = its sequential path."""
    cores = os.cpu_count() or 1
    best = 0
    for n in range(2, min(cores, frames) + 1):
        if frames % n == 0 and frames // n >= N_LOCAL // 2:
            best = n
    return best


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    frames = FRAMES_PER_GPU * args.gpus
    workers = ref_workers(frames)
    side = args.cpu_sample_hw
    fixed = cpu_fixed_cost(frames, workers)
    # a fixed 8x8 crop; only if K + W samples would run past ~5 minutes is it halved
    _, probe_wall = cpu_reference_sample(frames, side, workers, fixed)
    while side > 2 and probe_wall * (args.steps + args.warmup) > 300.0:
        side //= 2
        probe_wall = fixed + (probe_wall - fixed) / 4.0
    for _ in range(max(0, args.warmup - 1)):
        cpu_reference_sample(frames, side, workers, fixed)
    vals, walls = [], []
    for _ in range(args.steps):
        v, w = cpu_reference_sample(frames, side, workers, fixed)
        vals.append(v)
        walls.append(w)
    value = float(sum(vals) / len(vals))
    threads = max(workers, 1)
    sample = (f"reference execute_run (1 block, 1 step) on F={frames} frames of a {side}x{side} "
              f"crop of the 40x64 latent, C={C}, {'in-process clip-parallel x%d' % workers if workers else 'sequential'}; "
              f"fixed cost {fixed:.3f}s (1x1 crop run) subtracted, then frames/s scaled by "
              f"{H * W}/{side * side} positions")
    line = {"metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * sum(walls) / len(walls), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "impl": "reference",
            "config": workload_config(args.gpus, "f32"),
            "cpu_baseline": {"value": value, "unit": "frames/s", "cores": threads,
                             "host_cores": os.cpu_count(), "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(n: int, dtype: str) -> dict:
    return {"workload": "BASELINE configs[1] (N=1) / configs[2] (N>1): clip-parallel dual-scope "
                        "temporal block, 24 frames/GPU, 40x64 latent, C=640, 16 global frames",
            "frames": FRAMES_PER_GPU * n, "frames_per_gpu": FRAMES_PER_GPU, "height": H,
            "width": W, "channels": C, "taps": TAPS, "groups": GROUPS, "heads": HEADS,
            "n_local": N_LOCAL, "n_global": N_GLOBAL, "bias": BIAS, "t": T_STEP, "blocks": 1,
            "parallelism": f"clip-parallel x{n}",
            "executor": "C++ vinf_engine_forward_dist over NCCL (N>1); CUDA-graph replay of the block",
            "l2": "per-step working set ~1 GB >> 126 MB L2; the step's input is re-read cold",
            "dtype": dtype}


# ---- clocks ---------------------------------------------------------------------


class ClockSampler:
    """Samples SM clock + throttle reasons via NVML every 20 ms on a thread."""

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001
            pass

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksThrottleReasonSwPowerCap", 0x4),
            "hw_power_brake": getattr(nv, "nvmlClocksThrottleReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(s)}


# ---- our arm --------------------------------------------------------------------

def kernel_work(f_clip: int, dtype_bytes: int, split: bool = False, h: int = H, w: int = W, c: int = C,
                fused_o: bool = False):
    """Algorithmic work per launch for each kernel group: GEMM flops 2*M*N*K
    (x3 in the fp32 mode: every product runs as bf16 hi*hi + hi*lo + lo*hi on the tensor
    pipe, so that is the tensor work against the bf16 peak); bandwidth kernels their
    compulsory bytes (fp32 mode: Q/K/V and ctx as two bf16 planes = 4 B per element).
    fused_o (one head, engine.cpp fuse_o): the O projection is absorbed into V (W_vo = W_o W_v,
    a C^3 GEMM per step) and the attention core reads the residual and writes the block
    output instead of ctx (Q/K/V + residual in, y out)."""
    hw = h * w
    M = f_clip * hw
    E = hw * c
    s = dtype_bytes
    k = 3.0 if split else 1.0
    return {
        "conv_gemm": (k * 2.0 * M * c * TAPS * c, "tensor"),
        "qkv_gemm": (k * 2.0 * M * 3 * c * c, "tensor"),
        "o_gemm": (k * 2.0 * M * c * c, "tensor"),
        "kv_gemm_ctx": (None, "tensor"),
        "stub": (f_clip * E * (s + (2 * s if split else s)), "hbm"),  # fp32: x in; u (fp32) + hi/lo out
        "gn_stats": (((M + 31) // 32) * 2 * c * 4, "hbm"),
        "gn_apply": (f_clip * E * (s + 2 * s), "hbm") if split else (f_clip * E * (s + s), "hbm"),
        "gn_fold": (3 * c * c * (2 + 2) + 3 * c * 4, "hbm"),  # W read, W' + b' written
        "attn_core": (f_clip * E * s * 4, "hbm"),  # Q, K, V once + ctx write
        "wvo_gemm": (k * 2.0 * c * c * c, "tensor"),
    } if not fused_o else {
        "conv_gemm": (k * 2.0 * M * c * TAPS * c, "tensor"),
        "qkv_gemm": (k * 2.0 * M * 3 * c * c, "tensor"),
        "wvo_gemm": (k * 2.0 * c * c * c, "tensor"),
        "kv_gemm_ctx": (None, "tensor"),
        "stub": (f_clip * E * (s + (2 * s if split else s)), "hbm"),
        "gn_stats": (((M + 31) // 32) * 2 * c * 4, "hbm"),
        "gn_apply": (f_clip * E * (s + 2 * s), "hbm") if split else (f_clip * E * (s + s), "hbm"),
        "gn_fold": (3 * c * c * (2 + 2) + 3 * c * 4, "hbm"),
        # Q, K, V once + residual (bf16 raw u; fp32 GN output) + y (bf16; fp32)
        "attn_core": (f_clip * E * (s * 3 + (4 if split else s) * 2), "hbm"),
    }


def roofline_of(work: dict, stats: dict, tf: float, hbm: float, steps: int):
    """Per-kernel achieved rate and fraction of its bound, from per-kernel CUDA-event totals."""
    per = {}
    tot_all = sum(v[0] for v in stats.values()) or 1.0
    for k, (tot, cnt) in stats.items():
        row = {"ms_per_launch": tot / max(cnt, 1), "launches": cnt, "per_step_ms": tot / steps,
               "share": tot / tot_all}
        w_, bound = work.get(k, (None, None))
        if w_:
            ach = w_ / (row["ms_per_launch"] / 1000.0) / (1e12 if bound == "tensor" else 1e9)
            row.update(achieved=ach, unit="TFLOP/s" if bound == "tensor" else "GB/s",
                       frac=ach / (tf if bound == "tensor" else hbm), bound=bound)
        per[k] = row
    return per


class _Timer:
    """K steps between barrier + synchronize on both sides, CUDA events on the launching
    stream, the max over ranks; clocks sampled during the region."""

    def __init__(self, dev, local, world):
        self.dev, self.local, self.world = dev, local, world

    def barrier(self):
        import torch
        import torch.distributed as dist
        if self.world > 1:
            dist.barrier()
        torch.cuda.synchronize(self.dev)

    def run(self, step, steps, sample_clocks=True):
        import torch
        stream = torch.cuda.current_stream(self.dev)
        clocks = ClockSampler(self.local) if sample_clocks else None
        with (clocks or _Null()):
            self.barrier()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            for _ in range(steps):
                step()
            t1.record(stream)
            self.barrier()
        ms = max_over_ranks(t0.elapsed_time(t1), self.dev)
        return ms, (clocks.summary() if clocks else None)


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def _block_engine(en, ops, n, rank, dtype, dev, frames_per_gpu=FRAMES_PER_GPU, weight_seed=1):
    import torch  # noqa: F401
    F = frames_per_gpu * n
    desc = en.make_desc(F, n, rank, H, W, C, TAPS, GROUPS, HEADS, N_LOCAL, N_GLOBAL, BIAS,
                        T_STAR, 1e-5, 0.0, 1, dtype)
    eng = en.ClipEngine(en.Layout(desc), device=dev)
    eng.init_weights(weight_seed)
    # synthetic latent: this rank's frames of tensor_from_seed({F,H,W,C}, 0) (runner.cpp:59-60)
    fc = frames_per_gpu
    x = ops.tensor_from_seed((fc, H, W, C), 0, first_elem=rank * fc * H * W * C, dtype=dtype, device=dev)
    eng.x.copy_(x)
    return eng, x


def _profile(eng, step, steps, timer):
    """The same K steps again with CUDA events around every kernel group (vinf_engine_profile):
    they serialise the stream, so this run only gives the per-kernel breakdown."""
    import torch
    eng.profile(True)
    eng.kernel_stats()
    stream = torch.cuda.current_stream(timer.dev)
    timer.barrier()
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(steps):
        step()
    p1.record(stream)
    timer.barrier()
    stats = eng.kernel_stats()
    eng.profile(False)
    return stats, p0.elapsed_time(p1) / steps


def make_group(en, executor: str):
    """The clip-parallel executor of this rank: the C++ one over an NCCL communicator
    (default), or the Python stage loop over torch.distributed."""
    if executor == "native":
        from paper_2406_16260_b200.comm import NcclComm
        return en.CommGroup([NcclComm.create()])
    from paper_2406_16260_b200.transport import DistTransport
    return en.DistGroup(DistTransport())


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2406_16260_b200 import engine as en
    from paper_2406_16260_b200 import ops

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = max(world, 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1 or args.force_dist:
        if world == 1 and "MASTER_ADDR" not in os.environ:  # single-rank NCCL group (path check)
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", RANK="0", WORLD_SIZE="1")
        dist.init_process_group("nccl", device_id=dev)
        group = make_group(en, args.executor)
    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    es = 2 if dtype == torch.bfloat16 else 4
    fc = FRAMES_PER_GPU
    timer = _Timer(dev, local, world)
    stream = torch.cuda.current_stream(dev)

    eng, x_dev = _block_engine(en, ops, n, rank, dtype, dev)

    def step():
        en.forward(T_STEP, [eng], group)

    for _ in range(args.warmup):
        step()
    timer.barrier()

    # ---- timed region: K device-resident steps (value) ---------------------------
    # The engine's normal path (a single worker replays its CUDA graph; workers > 1 run
    # the staged loop with the exchanges). Per-kernel CUDA events are NOT recorded here.
    l0 = eng.launches()
    ms_max, clocks = timer.run(step, args.steps)
    launches = (eng.launches() - l0) // args.steps
    ms_per_step = ms_max / args.steps
    value = n * fc * args.steps / (ms_max / 1000.0)
    stats, profiled_ms_per_step = _profile(eng, step, args.steps, timer)

    # ---- e2e: host buffers in, host buffers out, through the public engine API ----
    # Two engines alternate steps; the upload of step j+1 (H2D stream) and the download of
    # step j-1 (D2H stream) overlap step j's kernels, so PCIe runs both directions while
    # the GPU computes. Every step still moves its whole clip in and its output out.
    eng2, _ = _block_engine(en, ops, n, rank, dtype, dev)
    engs = [eng, eng2]
    h_in = torch.empty((fc, H, W, C), dtype=dtype, pin_memory=True)
    h_in.copy_(x_dev.cpu())
    h_out = [torch.empty_like(h_in, pin_memory=True) for _ in range(2)]
    s_up, s_down = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    e_steps = max(4, min(args.steps, 200))  # the same K as the device-timed region

    def run_e2e(n_steps):
        ev = lambda: torch.cuda.Event()  # noqa: E731
        up_done, comp_done, down_done = {}, {}, {}
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(stream)

        def upload(j):
            e = engs[j % 2]
            s_up.wait_event(start)
            if j - 2 in comp_done:  # the engine's previous step has consumed its input
                s_up.wait_event(comp_done[j - 2])
            with torch.cuda.stream(s_up):
                e.x.copy_(h_in, non_blocking=True)
            up_done[j] = ev()
            up_done[j].record(s_up)

        upload(0)
        for j in range(n_steps):
            if j + 1 < n_steps:
                upload(j + 1)
            e = engs[j % 2]
            stream.wait_event(up_done[j])
            if j - 2 in down_done:  # its output buffer has been read back
                stream.wait_event(down_done[j - 2])
            en.forward(T_STEP, [e], group)
            comp_done[j] = ev()
            comp_done[j].record(stream)
            s_down.wait_event(comp_done[j])
            with torch.cuda.stream(s_down):
                h_out[j % 2].copy_(e.y, non_blocking=True)
            down_done[j] = ev()
            down_done[j].record(s_down)
        stream.wait_event(down_done[n_steps - 1])
        end.record(stream)
        return start, end

    run_e2e(3)
    timer.barrier()
    e0, e1 = run_e2e(e_steps)
    timer.barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1), dev)
    e2e_value = n * fc * e_steps / (e2e_ms / 1000.0)
    clip_bytes = fc * H * W * C * es
    # every step ran the same input: the host copies must equal the device result bitwise
    e2e_ok = bool(torch.equal(h_out[0], eng.y.cpu()) and torch.equal(h_out[1], eng.y.cpu()))
    del eng2, engs

    # ---- roofline of the dominant kernel (peaks chosen by the clocks of the region) ------
    hbm, tf_burst, tf_sus, src = peaks()
    tf, which, both = tensor_peak(clocks)
    fused_o = "o_gemm" not in stats  # engine.cpp fuse_o: the O projection absorbed into V
    work = kernel_work(fc, es, split=dtype == torch.float32, fused_o=fused_o)
    per_kernel = roofline_of(work, stats, tf, hbm, args.steps)
    dom = max(stats, key=lambda k: stats[k][0]) if stats else None
    roof = None
    if dom and per_kernel[dom].get("frac") is not None:
        pk = per_kernel[dom]
        roof = {"kernel": dom, "bound": pk["bound"], "achieved": pk["achieved"],
                "peak": tf if pk["bound"] == "tensor" else hbm, "unit": pk["unit"], "frac": pk["frac"],
                "traffic": None,
                "peak_source": (f"{src} bf16 {which} (SM clock held at max, no power cap)" if which == "burst"
                                else f"{src} bf16 sustained (clock below max or power capped)")
                if pk["bound"] == "tensor" else f"{src} HBM copy",
                "peaks": both, "work_per_launch": work[dom][0]}
    # DRAM traffic of the dominant kernel from the committed ncu --set full capture of this
    # workload (dram__bytes_read.sum + dram__bytes_write.sum per launch)
    if roof is not None and args.dtype == "bf16":
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                tr = json.load(f).get(roof["kernel"])
            if tr:
                roof["traffic"] = tr["dram_bytes"]
                roof["traffic_source"] = tr["source"]
        except (OSError, ValueError):
            pass
    # tensor work executed per step (fused: W_vo in place of the O GEMM); the reference's own
    # count (conv + Q/K/V + O projections) beside it
    flops_step = sum(work[k][0] for k in ("conv_gemm", "qkv_gemm", "o_gemm", "wvo_gemm") if k in work)
    ref_flops = sum(kernel_work(fc, es)[k][0] for k in ("conv_gemm", "qkv_gemm", "o_gemm"))
    floor = kernel_floor_us(fc, H, W, C, es, hbm, tf, fused_o=fused_o)
    block_roof = {"flops_per_step": flops_step, "reference_flops_per_step": ref_flops,
                  "o_projection": "absorbed into V (W_vo = W_o W_v each step)" if fused_o else "GEMM",
                  "achieved_tflops": flops_step / (ms_per_step / 1000.0) / 1e12,
                  "frac_of_tensor_peak": flops_step / (ms_per_step / 1000.0) / 1e12 / tf,
                  "tensor_peak": {"value": tf, "which": which, **both},
                  # per-kernel floor: each kernel at max(tensor time, HBM time) (kernel_floor_us)
                  "kernel_floor_us": sum(floor.values()),
                  "frac_of_kernel_floor": sum(floor.values()) / (ms_per_step * 1000.0),
                  "kernel_floor_parts_us": floor}

    # ---- fp32 mode (the reference's arithmetic, 1e-4 bar): same workload, timed ---------
    f32_rec = None
    if dtype == torch.bfloat16 and not args.no_f32:
        del eng
        torch.cuda.empty_cache()
        e32, _ = _block_engine(en, ops, n, rank, torch.float32, dev)

        def step32():
            en.forward(T_STEP, [e32], group)

        for _ in range(max(3, args.warmup)):
            step32()
        k32 = max(3, min(args.steps, 20))
        ms32, clk32 = timer.run(step32, k32)
        st32, _ = _profile(e32, step32, k32, timer)
        tf32, which32, _ = tensor_peak(clk32)
        w32 = kernel_work(fc, 4, split=True, fused_o="o_gemm" not in st32)
        pk32 = roofline_of(w32, st32, tf32, hbm, k32)
        f32_rec = {"value": n * fc * k32 / (ms32 / 1000.0), "unit": "frames/s",
                   "ms_per_step": ms32 / k32, "steps": k32,
                   "arithmetic": "bf16x3 split (hi*hi + hi*lo + lo*hi) on the tensor pipe, fp32 accumulate; "
                                 "parity bar 1e-4 normwise",
                   "tensor_peak": {"value": tf32, "which": which32},
                   "kernels": {k: {kk: v[kk] for kk in ("per_step_ms", "frac", "unit") if kk in v}
                               for k, v in pk32.items()},
                   "clocks": clk32}
        del e32
        torch.cuda.empty_cache()
    else:
        del eng

    # ---- configs[3]: the 2,300-frame VideoCrafter2-shaped stack over these N GPUs -----
    vc2_rec = None
    if not args.no_vc2:
        vc2_rec = measure_vc2(en, ops, n, rank, dtype, dev, group, timer, frames=2300,
                              steps=max(3, min(args.steps, 10)), warmup=2)

    cpu = None
    if rank == 0 and n == 1 and not args.no_cpu_baseline:
        try:
            side = args.cpu_sample_hw
            workers = ref_workers(fc)
            fixed = cpu_fixed_cost(fc, workers)
            v, wall = cpu_reference_sample(fc, side, workers, fixed)
            cpu = {"value": v, "unit": "frames/s", "cores": max(workers, 1), "host_cores": os.cpu_count(),
                   "kind": "reference",
                   "sample": f"reference execute_run, {'in-process clip-parallel x%d' % workers if workers else 'sequential'} "
                             f"(its most parallel form: no intra-op threading, F/N >= the 8-frame halo), F={fc}, "
                             f"{side}x{side} crop of 40x64, C={C}, 1 block 1 step, wall {wall:.2f}s minus "
                             f"fixed cost {fixed:.3f}s; frames/s scaled by {H * W}/{side * side} positions"}
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": "frames/s", "cores": 0, "host_cores": os.cpu_count(),
                   "kind": "reference", "sample": f"unavailable: {ex}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": n,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": args.dtype, "data": "synthetic (tensor_from_seed / build_model seeds 0/1)",
                "config": workload_config(n, args.dtype),
                "roofline": roof, "block_roofline": block_roof, "kernels": per_kernel,
                "kernel_timing": {"region": "second run of the same K steps with CUDA events around "
                                            "every kernel group (the headline region runs without "
                                            "them)", "profiled_ms_per_step": profiled_ms_per_step},
                "f32_mode": f32_rec,
                "vc2_stack_2300": vc2_rec,
                "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": clip_bytes,
                        "d2h_bytes_per_step": clip_bytes, "steps": e_steps,
                        "pipelining": "2 engines; H2D(j+1) and D2H(j-1) overlap step j",
                        "output_matches_device": e2e_ok},
                "gpu_launches": int(launches * args.steps), "clocks": clocks}
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()
    return 0


VC2_LEVELS = [(320, 40, 64), (640, 20, 32), (1280, 10, 16), (1280, 5, 8)]  # (C, H, W), SURVEY §8(a)


def measure_vc2(en, ops, n, rank, dtype, dev, group, timer, frames, steps, warmup):
    """BASELINE configs[3]: the VideoCrafter2-shaped temporal-layer stack, one dual-scope
    block per level (C, HxW) = (320, 40x64), (640, 20x32), (1280, 10x16), (1280, 5x8), over
    `frames` frames split into n clips (strong scaling: 2,300 over 8 GPUs = clips of 287/288
    frames, the uneven-clip extension). A step = every level's block over this GPU's clip,
    with the 3-step sync per level when n > 1."""
    import torch
    engines = []
    for li, (c, h, w) in enumerate(VC2_LEVELS):
        desc = en.make_desc(frames, n, rank, h, w, c, TAPS, GROUPS, HEADS, N_LOCAL, N_GLOBAL, BIAS,
                            T_STAR, 1e-5, 0.0, 1, dtype, uneven=frames % n != 0)
        lay = en.Layout(desc)
        fc = lay.f_clip
        e = en.ClipEngine(lay, device=dev)
        e.init_weights(1 + li)
        e.x.copy_(ops.tensor_from_seed((fc, h, w, c), li, first_elem=lay.start * h * w * c,
                                       dtype=dtype, device=dev))
        engines.append(e)
    stream = torch.cuda.current_stream(dev)

    def step():
        for e in engines:
            en.forward(T_STEP, [e], group)

    for _ in range(warmup):
        step()
    ms, clocks = timer.run(step, steps)
    # per-level split from a second pass with events between levels
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(engines) + 1)] for _ in range(steps)]
    timer.barrier()
    for k in range(steps):
        evs[k][0].record(stream)
        for li, e in enumerate(engines):
            en.forward(T_STEP, [e], group)
            evs[k][li + 1].record(stream)
    timer.barrier()
    level_ms = [sum(evs[k][li].elapsed_time(evs[k][li + 1]) for k in range(steps)) / steps
                for li in range(len(engines))]
    hbm, _, _, _ = peaks()
    tf, which, both = tensor_peak(clocks)
    es = 2 if dtype == torch.bfloat16 else 4
    k = 1.0 if dtype == torch.bfloat16 else 3.0
    fcs = [e.layout.f_clip for e in engines]
    # the engine absorbs the O projection into V for one head (engine.cpp fuse_o)
    fused = HEADS == 1 and os.environ.get("VINF_NO_FUSE_O", "0") in ("", "0")
    flops = [k * ((12.0 * fc * h * w * c * c + 2.0 * c ** 3) if fused else 14.0 * fc * h * w * c * c)
             for fc, (c, h, w) in zip(fcs, VC2_LEVELS)]
    floors = [sum(kernel_floor_us(fc, h, w, c, es, hbm, tf, fused_o=fused).values())
              for fc, (c, h, w) in zip(fcs, VC2_LEVELS)]
    levels = [{"channels": c, "height": h, "width": w, "frames_per_gpu": fc, "ms": m,
               "achieved_tflops": fl / (m / 1000.0) / 1e12, "frac_of_tensor_peak": fl / (m / 1000.0) / 1e12 / tf,
               "kernel_floor_ms": fu / 1000.0, "frac_of_kernel_floor": fu / 1000.0 / m}
              for fc, (c, h, w), m, fl, fu in zip(fcs, VC2_LEVELS, level_ms, flops, floors)]
    del engines
    torch.cuda.empty_cache()
    return {"workload": "BASELINE configs[3]: VideoCrafter2-shaped temporal stack, one dual-scope block per "
                        "level", "frames": frames, "n_gpus": n, "value": frames * steps / (ms / 1000.0),
            "unit": "frames/s", "scaling": "strong", "ms_per_step": ms / steps, "steps": steps,
            "clips": "uneven (floor(w*F/N) split)" if frames % n else "even",
            "levels": levels, "tensor_peak": {"value": tf, "which": which, **both},
            "block_roofline": {"flops_per_step": sum(flops),
                               "frac_of_tensor_peak": sum(flops) / (ms / steps / 1000.0) / 1e12 / tf,
                               "kernel_floor_ms": sum(floors) / 1000.0,
                               "frac_of_kernel_floor": sum(floors) / 1000.0 / (ms / steps)},
            "clocks": clocks}


def run_vc2(args):
    """--workload vc2: the configs[3] stack alone (--frames frames over this run's GPUs)."""
    import torch
    import torch.distributed as dist

    from paper_2406_16260_b200 import engine as en
    from paper_2406_16260_b200 import ops

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = max(world, 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        group = make_group(en, args.executor)
    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    rec = measure_vc2(en, ops, n, rank, dtype, dev, group, _Timer(dev, local, world), args.frames,
                      args.steps, args.warmup)
    if rank == 0:
        line = {"metric": METRIC, "value": rec["value"], "unit": "frames/s", "n_gpus": n,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": rec["ms_per_step"],
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": args.dtype, "data": "synthetic (tensor_from_seed / build_model seeds)",
                "config": {"workload": rec["workload"], "frames": args.frames,
                           "levels": [list(x) for x in VC2_LEVELS], "groups": GROUPS,
                           "n_local": N_LOCAL, "n_global": N_GLOBAL, "t": T_STEP,
                           "parallelism": f"clip-parallel x{n}", "clips": rec["clips"]},
                "block_roofline": rec["block_roofline"], "levels": rec["levels"], "clocks": rec["clocks"]}
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _stdout_for_result_only() -> None:
    """The driver reads ONE JSON line from stdout. Libraries may print there too (NCCL
    prints its version line to stdout when NCCL_DEBUG=WARN/VERSION), so route the process's
    fd 1 to stderr and keep a private handle on the real stdout for the result line."""
    global print
    real = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    builtin_print = print

    def _print(*a, **k):
        if "file" not in k:
            k["file"] = real
        builtin_print(*a, **k)

    print = _print  # noqa: A001


def main():
    args = parse()
    if args.impl == "ours":
        try:
            import torch
            visible = torch.cuda.device_count()
        except Exception:  # noqa: BLE001
            visible = 0
        argv = plan_launch(args.gpus, visible, os.environ, os.path.abspath(__file__), sys.argv[1:],
                           _free_port())
        if argv is not None:  # one process per GPU: re-run this command under torchrun
            os.execv(sys.executable, [sys.executable, *argv])
    _stdout_for_result_only()
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "vc2":
        return run_vc2(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
