cd $GRAFT_REPO_ROOT
for sp in 0 200 2000 20000; do for fz in 0 1; do echo -n "suspend $sp fuse $fz: "; env $( [ $fz = 1 ] && echo VINF_DIAG_FUSE=1 ) VINF_ATTN_SUSPEND=$sp timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 0 0; done; done
