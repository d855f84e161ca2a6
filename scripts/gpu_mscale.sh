# GEMM time vs M at the cfg2 O / QKV shapes (fixed per-launch overhead vs per-tile cost)
cd $GRAFT_REPO_ROOT
for m in 30720 61440 122880 245760; do
  timeout 300 python scripts/gemm_micro.py o$m=$m,640,640,1,1 q$m=$m,1920,640,1,0 c$m=$m,640,640,3,1 --flags=0,1
done
