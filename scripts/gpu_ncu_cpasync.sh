cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python scripts/attn_micro.py 288 40 64 320 1 16 16 0"
VINF_DIAG_FUSE=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention_core -s 1 -c 1 -o gpurun_out/prof_cpasync $CMD > gpurun_out/ncu_cpasync.log 2>&1; echo "ncu rc=$?"
