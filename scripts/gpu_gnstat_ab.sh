cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-f32 --no-vc2"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"colpart|group_fold" --csv --log-file gpurun_out/gn_launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-f32 --no-vc2 > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('value', round(d['value']), {k: round(v['ms_per_launch']*1000,1) for k,v in d['kernels'].items()})"
