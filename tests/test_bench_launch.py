"""bench.py's multi-GPU plumbing on CPU: `--gpus N` re-executes itself as N ranks under
torch.distributed.run (one process per GPU) and refuses to run on fewer visible GPUs than
requested; the timed region's max-over-ranks reduction over a real 2-rank gloo group."""
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_single_gpu_runs_in_process():
    assert bench.plan_launch(1, 1, {}, "bench.py", [], 1234) is None


def test_torchrun_rank_runs_in_process():
    assert bench.plan_launch(8, 8, {"WORLD_SIZE": "8"}, "bench.py", [], 1234) is None
    with pytest.raises(SystemExit):
        bench.plan_launch(4, 8, {"WORLD_SIZE": "8"}, "bench.py", [], 1234)


def test_too_few_gpus_fails_loudly():
    with pytest.raises(SystemExit, match="only 1 CUDA device"):
        bench.plan_launch(2, 1, {}, "bench.py", ["--gpus", "2"], 1234)
    with pytest.raises(SystemExit):
        bench.plan_launch(1, 0, {}, "bench.py", [], 1234)


def test_multi_gpu_reexecs_under_torchrun():
    argv = bench.plan_launch(4, 8, {}, "/x/bench.py", ["--gpus", "4", "--steps", "5"], 29555)
    assert argv[:2] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in argv and "--master-addr=127.0.0.1" in argv
    assert "--master-port=29555" in argv
    assert argv[-5:] == ["/x/bench.py", "--gpus", "4", "--steps", "5"]


def test_bench_gpus2_on_cpu_host_errors():
    # the real entry point: no CUDA device here, so --gpus 2 must exit non-zero, not measure 1
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "visible" in r.stderr
    assert r.stdout.strip() == ""


_WORKER = r'''
import os, sys
sys.path.insert(0, sys.argv[1])
import torch.distributed as dist
import bench
dist.init_process_group("gloo")
r = dist.get_rank()
v = bench.max_over_ranks(10.0 + r, device="cpu")
with open(os.path.join(sys.argv[2], f"rank{r}.txt"), "w") as f:  # ranks share one stdout pipe
    f.write(f"MAX {r} {v}")
dist.destroy_process_group()
'''


def test_max_over_ranks_gloo_world2(tmp_path):
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    script = tmp_path / "w.py"
    script.write_text(_WORKER)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", f"--master-port={port}", str(script), ROOT, str(tmp_path)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    outs = sorted((tmp_path / f"rank{i}.txt").read_text() for i in range(2))
    assert outs == ["MAX 0 11.0", "MAX 1 11.0"]
