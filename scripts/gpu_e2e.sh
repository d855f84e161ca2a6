cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --steps 100 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench.json'))
print("value", round(d["value"]), "ms/step", round(d["ms_per_step"],4), "e2e", d["e2e"], "cpu", d["cpu_baseline"], "clocks", d["clocks"], "launches", d["gpu_launches"])
print("roofline", d["roofline"]); print("block", d["block_roofline"])
PY
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --force-dist > gpurun_out/bench_dist.json 2> gpurun_out/bench_dist.err; echo "bench force-dist rc=$?"; tail -3 gpurun_out/bench_dist.err
python -c "import json; d=json.load(open('gpurun_out/bench_dist.json')); print('dist value', round(d['value']), d['e2e']['output_matches_device'])"
timeout 900 torchrun --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_torchrun.json 2> gpurun_out/bench_torchrun.err; echo "torchrun rc=$?"; tail -2 gpurun_out/bench_torchrun.err
timeout 600 python bench.py --dtype f32 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_f32.json 2> gpurun_out/bench_f32.err; echo "f32 rc=$?"; tail -2 gpurun_out/bench_f32.err
python -c "import json; d=json.load(open('gpurun_out/bench_f32.json')); print('f32 value', round(d['value']), 'ms', d['ms_per_step']); [print(' ', k, round(v['ms_per_launch']*1000,1)) for k,v in d['kernels'].items()]"
