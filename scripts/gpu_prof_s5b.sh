cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for fo in 0 1; do echo "== VINF_NO_FUSE_O=$fo"; VINF_NO_FUSE_O=$fo timeout 300 python scripts/level_profile.py 2304 40 64 320 3 2>&1 | tail -9; done
for nw in "2 0" "8 3"; do echo "== worker $nw"; timeout 300 python scripts/worker_profile.py $nw 10 2>&1 | tail -10; done
