cd $GRAFT_REPO_ROOT
for fs in 0 1; do for lo in 0 1 3; do echo -n "fullslots $fs fuse lo $lo: "; env $( [ $fs = 1 ] && echo VINF_ATTN_FULLSLOTS=1 ) VINF_DIAG_FUSE=1 VINF_ATTN_LOAD_ONLY=$lo VINF_ATTN_IMPL=tma timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 0 0; done; done
