cd $GRAFT_REPO_ROOT
for l in "2300 40 64 320" "2300 20 32 640" "2300 10 16 1280" "2300 5 8 1280"; do timeout 300 python scripts/level_profile.py $l 5 2>&1 | tail -10; done
