# main loop (nostore=1) vs full GEMM for the single-CTA and the CTA-pair kernels at the bench shapes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/gemm_micro.py conv qkv o 2>&1 | tee gpurun_out/micro_single.log
VINF_GEMM_PAIR=1 timeout 300 python scripts/gemm_micro.py conv qkv o 2>&1 | tee gpurun_out/micro_pair.log
for bn in 256 192 160; do VINF_GEMM_PAIR=1 VINF_GEMM_BN=$bn timeout 300 python scripts/gemm_micro.py qkv o 2>&1 | sed "s/^/pair bn=$bn /"; done
