cd $GRAFT_REPO_ROOT
for rows in 48 64; do for nw in "8 3" "4 1"; do echo -n "cw_rows $rows worker $nw: "; VINF_ATTN_CW_ROWS=$rows timeout 300 python scripts/worker_profile.py $nw 10 2>&1 | grep -E "attn_core|us/step \(" | tr '\n' ' '; echo; done
echo -n "cw_rows $rows F=288 C=320: "; VINF_ATTN_CW_ROWS=$rows timeout 60 python scripts/attn_micro.py 288 40 64 320 1 16 16 0 0
echo -n "cw_rows $rows F=288 C=640 20x32: "; VINF_ATTN_CW_ROWS=$rows timeout 60 python scripts/attn_micro.py 288 20 32 640 1 16 16 0 0
done
