# Same-box A/B of two source trees on one engine shape (level_profile.py): ./ against $1
# usage: bash scripts/gpu_ab_level.sh OLD "F H W C" [rounds]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
OLD=$1; SHAPE=$2; R=${3:-2}
for i in $(seq 1 $R); do
  for t in . $OLD; do
    echo "== $t"
    (cd $t && timeout 300 python scripts/level_profile.py $SHAPE 3)
  done
done
