cd $GRAFT_REPO_ROOT
for lo in 1 2; do VINF_ATTN_IMPL=tma VINF_ATTN_LOAD_ONLY=$lo timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 0 0; done
