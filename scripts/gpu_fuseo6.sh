cd $GRAFT_REPO_ROOT
for lo in 0 1 3; do echo -n "fuse lo $lo: "; VINF_DIAG_FUSE=1 VINF_ATTN_LOAD_ONLY=$lo VINF_ATTN_IMPL=tma timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 0 0; done
bash scripts/gpu_ab_env.sh "VINF_NO_FUSE_O=1" "VINF_NO_FUSE_O=0" 2
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
