# round 2: new TMA attention core -- parity suite, then bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -4 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_gpu.log | grep -v "^$" | tail -25
timeout 600 python bench.py --steps 50 --warmup 5 --no-vc2 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench.json'))
print("value", round(d["value"]), "ms/step", round(d["ms_per_step"],4), "e2e", round(d["e2e"]["value"]), "clocks", d["clocks"])
for k,v in d["kernels"].items(): print(f"  {k:12s} {v['ms_per_launch']*1000:8.1f} us  {v.get('achieved',0):8.1f} {v.get('unit','')}  frac {v.get('frac',0):.3f}")
f=d.get("f32_mode") or {}
print("f32", f.get("value"), {k: round(v["per_step_ms"]*1000,1) for k,v in (f.get("kernels") or {}).items()})
PY
tail -3 gpurun_out/bench.err
