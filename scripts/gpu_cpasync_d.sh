cd $GRAFT_REPO_ROOT
for fz in 0 1; do for args in "288 40 64 320 1 16 16 0" "2304 40 64 320 1 16 16 0" "288 20 32 640 1 16 16 0"; do echo -n "fuse $fz $args: "; env $( [ $fz = 1 ] && echo VINF_DIAG_FUSE=1 ) VINF_ATTN_IMPL=cpasync timeout 120 python scripts/attn_micro.py $args 0; done; done
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
