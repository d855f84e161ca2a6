cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest_fuseo.log
tail -12 gpurun_out/pytest_fuseo.log
bash scripts/gpu_ab_env.sh "VINF_NO_FUSE_O=1" "VINF_NO_FUSE_O=0" 2
