cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
bash scripts/gpu_ab_env.sh "VINF_QKV_NATURAL=1" "VINF_NO_FUSE_O=0" 3
