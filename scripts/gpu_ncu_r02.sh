# round-2 ncu evidence: launch list of the bench step + one full capture of each kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-f32 --no-vc2"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc|attention_core|group_fold|colpart|stub" -s 6 -c 7 -o gpurun_out/r02_prof $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
