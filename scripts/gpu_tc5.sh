cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_attention_impl.py -m gpu -q -p no:cacheprovider 2>&1 | tail -15
for impl in tma tc5; do for fz in 0 1; do echo -n "$impl fuse $fz: "; env $( [ $fz = 1 ] && echo VINF_DIAG_FUSE=1 ) VINF_ATTN_IMPL=$impl timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 0 0; done; done
