# Same-box A/B of two source trees: ./ (new) against $1 (an older worktree with its own built .so)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
OLD=$1; R=${2:-3}
for i in $(seq 1 $R); do
  for t in . $OLD; do
    (cd $t && timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > $GRAFT_REPO_ROOT/gpurun_out/abt.json 2>/dev/null)
    python -c "import json; d=json.load(open('gpurun_out/abt.json')); k=d['kernels']; print('$t', round(d['ms_per_step']*1000,1), 'us', d['clocks']['sm_mhz'], ' '.join(f'{n}={v[\"ms_per_launch\"]*1000:.1f}' for n,v in k.items()))"
  done
done
