cd $GRAFT_REPO_ROOT
for lo in 0 3; do VINF_ATTN_LOAD_ONLY=$lo VINF_ATTN_IMPL=tma timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 0 0; done
timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 1 0
timeout 600 python -m pytest tests -m gpu -x -q -k "attention or baseline or parity" 2>&1 | tail -3
