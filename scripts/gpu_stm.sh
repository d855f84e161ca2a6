cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for fz in 0 1; do for lo in 0 3; do echo -n "fuse $fz lo $lo: "; env $( [ $fz = 1 ] && echo VINF_DIAG_FUSE=1 ) VINF_ATTN_LOAD_ONLY=$lo timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 0 0; done; done
bash scripts/gpu_ab_env.sh "VINF_NO_FUSE_O=0" "VINF_NO_FUSE_O=0" 1
