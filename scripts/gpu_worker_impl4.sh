cd $GRAFT_REPO_ROOT
for nw in "2 0" "4 1" "8 3"; do echo -n "worker $nw: "; timeout 300 python scripts/worker_profile.py $nw 10 2>&1 | grep -E "attn_core|us/step \(" | tr '\n' ' '; echo; done
echo -n "F=288 C=320: "; timeout 60 python scripts/attn_micro.py 288 40 64 320 1 16 16 0 0
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
