# GPU tests + bench + ncu evidence (launch list of the bench command, full capture of the top kernels)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 100 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench.json'))
print("value", round(d["value"]), "ms/step", round(d["ms_per_step"],4), "e2e", round(d["e2e"]["value"]), "clocks", d["clocks"])
for k,v in d["kernels"].items(): print(f"  {k:12s} {v['ms_per_launch']*1000:8.1f} us  share {v['share']:.3f}  {v.get('achieved',0):8.1f} {v.get('unit','')}  frac {v.get('frac',0):.3f}")
PY
CMD="python bench.py --steps 3 --warmup 2 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 300 $CMD > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc|attention_core|group_apply|group_fold|stub|colpart|colseg" -s 8 -c 9 -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
ls -la gpurun_out
