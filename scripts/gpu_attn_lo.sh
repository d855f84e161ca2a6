cd $GRAFT_REPO_ROOT
for cfg in "4 3" "4 4" "4 2" "8 2" "8 1"; do set -- $cfg
 for lo in 0 3; do echo -n "warps $1 ctas $2 lo $lo: "; VINF_ATTN_WARPS=$1 VINF_ATTN_CTAS=$2 VINF_ATTN_LOAD_ONLY=$lo VINF_ATTN_IMPL=tma timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 0 0; done
done
