# round 2: C++ executor tests, single-rank NCCL bench path, ncu launch list + attention-core capture
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_executor.py -x -q > gpurun_out/pytest_exec.log 2>&1; echo "exec tests rc=$?"; tail -15 gpurun_out/pytest_exec.log
timeout 300 python bench.py --force-dist --steps 50 --warmup 5 --no-f32 --no-vc2 --no-cpu-baseline > gpurun_out/bench_dist1.json 2> gpurun_out/bench_dist1.err; echo "dist1 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_dist1.json')); print('force-dist value', round(d['value']), 'ms', d['ms_per_step'])"
tail -3 gpurun_out/bench_dist1.err
CMD="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-f32 --no-vc2"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attention_core|gemm_tc" -s 4 -c 4 -o gpurun_out/prof_r02 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
ls gpurun_out
