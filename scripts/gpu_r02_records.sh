# round 2 records: configs[4] sweep, Table-3 sync ablation (in-process workers), worker profiles
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/bench_sweep.py --steps 10 --out gpurun_out/r02_cfg5_sweep.json > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"; tail -3 gpurun_out/sweep.log
timeout 900 python scripts/table3.py --workers 1 2 4 8 --steps 5 --out gpurun_out/r02_table3.json > gpurun_out/table3.log 2>&1; echo "table3 rc=$?"; tail -5 gpurun_out/table3.log
for nw in "1 0" "2 0" "2 1" "8 0" "8 3" "8 7"; do timeout 120 python scripts/worker_profile.py $nw 10 2>&1 | tail -12; done > gpurun_out/worker_profile.log; echo "wp rc=$?"; cat gpurun_out/worker_profile.log | head -60
