cd $GRAFT_REPO_ROOT
for qf in 1 2; do for lo in 0 1; do echo -n "qfeed $qf lo $lo: "; VINF_ATTN_QFEED=$qf VINF_ATTN_LOAD_ONLY=$lo VINF_ATTN_IMPL=tma timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 0 0; done; done
for qf in 0; do echo -n "C=320 F=2304 qfeed $qf: "; VINF_ATTN_QFEED=$qf VINF_ATTN_IMPL=tma timeout 60 python scripts/attn_micro.py 2304 40 64 320 1 16 16 0 0; done
timeout 600 python -m pytest tests -m gpu -x -q -k "attention or baseline or parity" 2>&1 | tail -3
