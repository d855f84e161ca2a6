cd $GRAFT_REPO_ROOT
for fz in 0 1; do echo -n "f32 cfg2 fuse $fz: "; env $( [ $fz = 1 ] && echo VINF_DIAG_FUSE=1 ) timeout 120 python scripts/attn_micro.py 24 40 64 640 1 16 16 1 0; done
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-vc2 > gpurun_out/b_f32.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/b_f32.json')); print(round(d['value']), round(d['f32_mode']['value']), round(d['f32_mode']['ms_per_step']*1000,1), d['f32_mode']['kernels']['attn_core'])"
