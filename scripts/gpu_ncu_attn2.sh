# one full capture of the attention core (TMA version) inside the bench's step
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD2="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-f32 --no-vc2"
timeout 300 $CMD2 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attention_core|group_fold|colpart" -s 3 -c 3 -o gpurun_out/prof_attn_tma $CMD2 > gpurun_out/ncu_attn.log 2>&1; echo "ncu rc=$?"
