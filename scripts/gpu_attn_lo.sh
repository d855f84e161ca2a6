cd $GRAFT_REPO_ROOT
for impl in tma cpasync; do
  echo "== $impl"
  for case in "24 40 64 640 1 16 16 0" "288 40 64 320 1 16 16 0" "288 40 64 640 1 16 64 0" "24 40 64 640 1 16 16 1" "288 40 64 320 1 16 16 1" "96 20 32 640 1 16 16 0" "288 10 16 1280 1 16 16 0"; do
   VINF_ATTN_IMPL=$impl timeout 60 python scripts/attn_micro.py $case 0
  done
done
