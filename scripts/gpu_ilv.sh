cd $GRAFT_REPO_ROOT
for ilv in 0 1; do for lo in 0 1 3; do echo -n "ilv $ilv lo $lo: "; VINF_ATTN_ILV=$ilv VINF_ATTN_LOAD_ONLY=$lo VINF_ATTN_IMPL=tma timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 0 0; done; done
for ilv in 0 1; do echo -n "F=288 C=320 tma ilv $ilv: "; VINF_ATTN_ILV=$ilv VINF_ATTN_IMPL=tma timeout 60 python scripts/attn_micro.py 288 40 64 320 1 16 16 0 0; done
for ilv in 0 1; do echo -n "cfg2 f32 tma ilv $ilv: "; VINF_ATTN_ILV=$ilv VINF_ATTN_IMPL=tma timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 1 0; done
timeout 600 python -m pytest tests -m gpu -x -q -k "attention or baseline or parity" 2>&1 | tail -3
