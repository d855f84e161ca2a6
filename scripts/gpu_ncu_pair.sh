# ncu --set full of the single-CTA and CTA-pair GEMM main loops (QKV shape, no epilogue traffic)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python scripts/gemm_micro.py qkv --once --flags=1"
timeout 300 $CMD && VINF_GEMM_PAIR=1 timeout 300 $CMD && \
timeout 900 ncu --set full --clock-control none -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/qkv_single $CMD > gpurun_out/ncu_s.log 2>&1; echo "single rc=$?"
VINF_GEMM_PAIR=1 timeout 900 ncu --set full --clock-control none -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/qkv_pair $CMD > gpurun_out/ncu_p.log 2>&1; echo "pair rc=$?"
