cd $GRAFT_REPO_ROOT
for i in 1 2; do VINF_ATTN_IMPL=tma timeout 60 python scripts/attn_micro.py 24 40 64 640 1 16 16 0 0; done
timeout 300 python -m pytest tests/test_cpp_mirror.py -q -x 2>&1 | tail -2
