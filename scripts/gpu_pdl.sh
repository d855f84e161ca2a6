cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in "" 1; do
  VINF_NO_PDL=$v timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_pdl$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/bench_pdl$v.json')); print('NO_PDL=$v', round(d['value']), round(d['ms_per_step']*1000,1), 'us', d['clocks'])"
done
python scripts/graph_vs_profile.py 2>&1 | tail -4
