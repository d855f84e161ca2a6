cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/attn_micro.py 2>&1 | tee gpurun_out/attn_micro.log
