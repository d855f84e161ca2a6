cd $GRAFT_REPO_ROOT
for w in 4 8; do for lo in 0 1 3; do echo -n "warps $w fused lo $lo: "; VINF_ATTN_WARPS=$w VINF_DIAG_FUSE=1 VINF_ATTN_LOAD_ONLY=$lo timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 0 0; done; done
bash scripts/gpu_ab_env.sh "VINF_ATTN_WARPS=4" "VINF_ATTN_WARPS=8" 2
