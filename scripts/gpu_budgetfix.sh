cd $GRAFT_REPO_ROOT
for args in "24 40 64 640 1 16 16 0" "288 40 64 320 1 16 16 0" "24 40 64 640 1 16 16 1" "96 20 32 640 1 16 16 0" "288 10 16 1280 1 16 16 0"; do echo -n "$args: "; VINF_ATTN_IMPL=tma timeout 60 python scripts/attn_micro.py $args 0; done
echo -n "fused cfg2: "; VINF_DIAG_FUSE=1 VINF_ATTN_IMPL=tma timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 0 0
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
bash scripts/gpu_ab_env.sh "VINF_NO_FUSE_O=1" "VINF_NO_FUSE_O=0" 2
