cd $GRAFT_REPO_ROOT
for bo in 0 20 100 500; do for fz in 0 1; do echo -n "backoff $bo fuse $fz: "; env $( [ $fz = 1 ] && echo VINF_DIAG_FUSE=1 ) VINF_ATTN_BACKOFF=$bo timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 0 0; done; done
