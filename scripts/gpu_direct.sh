cd $GRAFT_REPO_ROOT
M=$((2304*40*64))
for i in 1 2; do timeout 300 python scripts/gemm_micro.py qkv qkv320=$M,960,320,1,0 --flags=0,128,1; done
