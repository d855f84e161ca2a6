cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/gemm_micro.py 2>&1 | tail -12
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench.json'))
print("value", round(d["value"]), "ms/step", round(d["ms_per_step"],4), "e2e", round(d["e2e"]["value"]), "clocks", d["clocks"])
for k,v in d["kernels"].items(): print(f"  {k:12s} {v['ms_per_launch']*1000:8.1f} us  share {v['share']:.3f}  {v.get('achieved',0):8.1f} {v.get('unit','')}  frac {v.get('frac',0):.3f}")
PY
