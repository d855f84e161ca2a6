cd $GRAFT_REPO_ROOT
bash scripts/gpu_ab_env.sh "VINF_WVO_INLINE=1" "VINF_NO_FUSE_O=0" 3
