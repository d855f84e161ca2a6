cd $GRAFT_REPO_ROOT
for fo in 0 1; do echo "== VINF_NO_FUSE_O=$fo"; VINF_NO_FUSE_O=$fo timeout 300 python scripts/level_profile.py 2304 40 64 320 3 2>&1 | tail -9; done
for nw in "2 0" "8 3"; do echo "== worker $nw"; timeout 300 python scripts/worker_profile.py $nw 10 2>&1 | tail -12; done
