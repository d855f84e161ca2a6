cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python scripts/attn_micro.py 24 40 64 640 1 16 16 0"
VINF_ATTN_IMPL=tc5 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention_tc5 -s 1 -c 1 -o gpurun_out/prof_tc5 $CMD > gpurun_out/ncu_tc5.log 2>&1; echo "ncu rc=$?"
