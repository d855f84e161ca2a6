# Same-box A/B of an environment switch: alternating runs of the headline bench.
# usage: bash scripts/gpu_ab.sh VAR [rounds]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
VAR=$1; R=${2:-3}
for i in $(seq 1 $R); do
  for v in "" 1; do
    env ${v:+$VAR=${VAL:-1}} timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/ab_$v.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); k=d['kernels']; print('$VAR=${v:-0}', round(d['ms_per_step']*1000,1), 'us', d['clocks']['sm_mhz'], ' '.join(f'{n}={v[\"ms_per_launch\"]*1000:.1f}' for n,v in k.items()))"
  done
done
