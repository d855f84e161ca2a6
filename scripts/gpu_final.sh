# end-of-session evidence: GPU tests, smoke, headline bench, VC2 stack, ncu launch list + full capture
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_profile.sh
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --workload vc2 --steps 5 --warmup 3 > gpurun_out/vc2.json 2> gpurun_out/vc2.err; echo "vc2 rc=$?"
