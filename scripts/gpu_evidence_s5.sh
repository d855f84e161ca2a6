# session-5 evidence: default bench line, launch list of the bench step, one ncu --set full
# capture of each kernel of a step, the reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/s5_bench.json 2> gpurun_out/s5_bench.err; echo "bench rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-f32 --no-vc2"
timeout 300 $CMD > gpurun_out/s5_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s5_launches.csv $CMD > gpurun_out/s5_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc|attention_core|group_fold|colpart|stub" -s 14 -c 7 -o gpurun_out/s5_prof $CMD > gpurun_out/s5_ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s5_ref.json 2> gpurun_out/s5_ref.err; echo "ref rc=$?"
