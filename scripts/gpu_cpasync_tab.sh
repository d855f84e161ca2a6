cd $GRAFT_REPO_ROOT
for args in "288 40 64 320 1 16 16 0" "2304 40 64 320 1 16 16 0" "288 20 32 640 1 16 16 0"; do echo -n "fuse $args: "; VINF_DIAG_FUSE=1 VINF_ATTN_IMPL=cpasync timeout 120 python scripts/attn_micro.py $args 0; done
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python scripts/level_profile.py 2304 40 64 320 3 2>&1 | tail -9
