cd $GRAFT_REPO_ROOT
VINF_ATTN_IMPL=rows VINF_ATTN_LOAD_ONLY=1 timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 0 0
VINF_ATTN_IMPL=rows timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 0 0
