cd $GRAFT_REPO_ROOT
for bn in 0 192 256; do
VINF_GEMM_BN=$bn timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-f32 --no-vc2 > gpurun_out/b$bn.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b$bn.json')); print('BN $bn', round(d['value']), {k: round(v['ms_per_launch']*1000,1) for k,v in d['kernels'].items()})"
done
