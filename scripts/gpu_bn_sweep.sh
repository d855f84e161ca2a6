# block-N sweep of the cfg2 GEMMs (gemm_micro), default pick first
cd $GRAFT_REPO_ROOT
for r in 1 2; do
timeout 300 python scripts/gemm_micro.py conv o --once
for bn in 160 192 256; do VINF_GEMM_BN=$bn timeout 300 python scripts/gemm_micro.py conv o --once | sed "s/^/bn=$bn /"; done
done
