cd $GRAFT_REPO_ROOT
for nw in "2 0" "8 3" "4 1"; do echo -n "auto worker $nw: "; timeout 300 python scripts/worker_profile.py $nw 10 2>&1 | grep -E "attn_core|us/step \(" | tr '\n' ' '; echo; done
for nw in "2 0" "4 1"; do echo -n "cpasync worker $nw: "; VINF_ATTN_IMPL=cpasync timeout 300 python scripts/worker_profile.py $nw 10 2>&1 | grep -E "attn_core|us/step \(" | tr '\n' ' '; echo; done
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
