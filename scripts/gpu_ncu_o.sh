cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/gemm_micro.py conv qkv o > gpurun_out/micro.log 2>&1; cat gpurun_out/micro.log
SHAPE=o bash scripts/gpu_ncu_gemm.sh
