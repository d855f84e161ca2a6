cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 0 1; do
  echo "== VINF_GEMM_PAIR=$v"
  VINF_GEMM_PAIR=$v timeout 300 python scripts/gemm_micro.py conv qkv o 2>&1 | tail -6
done
VINF_GEMM_PAIR=1 timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
VINF_GEMM_PAIR=1 timeout 300 python scripts/diag_gemm_det.py 2>&1 | tail -5
