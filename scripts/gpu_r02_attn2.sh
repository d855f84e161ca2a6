cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CTAS="0 4" bash scripts/gpu_attn_micro.sh
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_gpu.log | grep -v "^$" | tail -4
