# GroupNorm folding A/B: GPU tests (fold on), then bench with and without the fold.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for v in "" 1; do
  VINF_NO_GN_FOLD=$v timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_fold$v.json 2>gpurun_out/bench_fold$v.err
  python -c "import json; d=json.load(open('gpurun_out/bench_fold$v.json')); print('NO_FOLD=$v', round(d['value']), round(d['ms_per_step']*1000,1), 'us', d['clocks'], d.get('kernel_timing'))"
done
