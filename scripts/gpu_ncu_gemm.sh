cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SHAPE=${SHAPE:-qkv}
CMD="python scripts/gemm_micro.py $SHAPE --once"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && cat gpurun_out/plain.log && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/gemm_$SHAPE $CMD > gpurun_out/ncu_gemm.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_gemm.log
