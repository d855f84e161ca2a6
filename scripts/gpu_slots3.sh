cd $GRAFT_REPO_ROOT
for fz in 0 1; do for fs in 0 1; do for lo in 0 1 3; do echo -n "fuse $fz fullslots $fs lo $lo: "; env $( [ $fs = 1 ] && echo VINF_ATTN_FULLSLOTS=1 ) $( [ $fz = 1 ] && echo VINF_DIAG_FUSE=1 ) VINF_ATTN_LOAD_ONLY=$lo VINF_ATTN_IMPL=tma timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 0 0; done; done; done
for args in "288 40 64 320 1 16 16 0" "24 40 64 640 1 16 16 1" "96 20 32 640 1 16 16 0"; do echo -n "$args: "; VINF_ATTN_IMPL=tma timeout 60 python scripts/attn_micro.py $args 0; done
