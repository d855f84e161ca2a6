cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in ${CTAS:-0}; do
  echo "== VINF_ATTN_CTAS=$c"
  VINF_ATTN_CTAS=$c timeout 120 python -X faulthandler scripts/attn_micro.py > gpurun_out/attn_micro_$c.log 2>&1; echo "micro rc=$?"; grep -v "read stream" gpurun_out/attn_micro_$c.log | tail -12
done
