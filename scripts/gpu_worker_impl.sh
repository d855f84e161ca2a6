cd $GRAFT_REPO_ROOT
for impl in tma cpasync; do for nw in "2 0" "8 3"; do echo -n "$impl worker $nw: "; VINF_ATTN_IMPL=$impl timeout 300 python scripts/worker_profile.py $nw 10 2>&1 | grep -E "attn_core|us/step \(" | tr '\n' ' '; echo; done; done
