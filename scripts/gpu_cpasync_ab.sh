cd $GRAFT_REPO_ROOT
for i in 1 2; do for old in 0 1; do for args in "288 40 64 320 1 16 16 0" "2304 40 64 320 1 16 16 0"; do echo -n "old $old $args: "; env $( [ $old = 1 ] && echo VINF_TMP_OLDSMX=1 ) VINF_ATTN_IMPL=cpasync timeout 120 python scripts/attn_micro.py $args 0; done; done; done
