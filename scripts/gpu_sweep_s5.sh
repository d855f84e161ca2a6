cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python scripts/bench_sweep.py --out gpurun_out/cfg5_sweep_s5.json > gpurun_out/sweep_s5.log 2>&1; echo "sweep rc=$?"
timeout 1200 python scripts/table3.py --out gpurun_out/table3_s5.json > gpurun_out/table3_s5.log 2>&1; echo "table3 rc=$?"
tail -5 gpurun_out/table3_s5.log
