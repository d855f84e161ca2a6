cd $GRAFT_REPO_ROOT
bash scripts/gpu_ab_env.sh "VINF_NO_FUSE_O=1" "VINF_NO_FUSE_O=0" 2
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
