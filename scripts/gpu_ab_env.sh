# Same-box A/B of two environment settings on the headline bench: bash scripts/gpu_ab_env.sh "A=1 B=2" "C=1" [rounds]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
R=${3:-2}
for i in $(seq 1 $R); do
  for cfg in "$1" "$2"; do
    env $cfg timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/abe.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/abe.json')); k=d['kernels']; print('[$cfg]', round(d['ms_per_step']*1000,1), 'us', d['clocks']['sm_mhz'], ' '.join(f'{n}={v[\"ms_per_launch\"]*1000:.1f}' for n,v in k.items()))"
  done
done
