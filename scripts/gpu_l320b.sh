cd $GRAFT_REPO_ROOT
timeout 300 python scripts/level_profile.py 2304 40 64 320 3 2>&1
for impl in tma cpasync; do VINF_ATTN_IMPL=$impl timeout 120 python scripts/attn_micro.py 2304 40 64 320 1 16 16 0 0; done
