# QKV epilogue cost split: full (0), no global traffic (1), staged but no TMA store (16), convert only (32)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M=$((2304*40*64))
for r in 1 2; do
timeout 300 python scripts/gemm_micro.py qkv --flags=0,128,16 2>&1
timeout 300 python scripts/gemm_micro.py qkv320=$M,960,320,1,0 --flags=0,128,16 2>&1
done | tee gpurun_out/epi_diag.log
