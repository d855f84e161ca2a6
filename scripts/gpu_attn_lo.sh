cd $GRAFT_REPO_ROOT
for pm in 0 3; do VINF_ATTN_IMPL=tma timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 0 $pm; done
VINF_ATTN_LOAD_ONLY=1 timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 0 3
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error" gpurun_out/pytest_gpu.log | tail -5
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-f32 --no-vc2 > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('value', round(d['value']), round(d['ms_per_step']*1000,1), {k: round(v['ms_per_launch']*1000,1) for k,v in d['kernels'].items()})"
