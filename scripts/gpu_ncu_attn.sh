cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
# one full capture of the attention core inside the bench's step (variant from the env)
CMD2="python bench.py --steps 3 --warmup 2 --no-cpu-baseline"
timeout 300 $CMD2 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attention_core" -s 2 -c 1 -o gpurun_out/prof_attn_${TAG:-x} $CMD2 > gpurun_out/ncu_attn.log 2>&1; echo "ncu rc=$?"
