cd $GRAFT_REPO_ROOT
for pm in 0 2 3; do
VINF_ATTN_LOAD_ONLY=1 timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 0 $pm
VINF_ATTN_LOAD_ONLY=1 timeout 60 python scripts/attn_micro.py 288 40 64 320 1 16 16 0 $pm
done
for c in 2 4; do
VINF_ATTN_CTAS=$c VINF_ATTN_LOAD_ONLY=1 timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 0 3
done
