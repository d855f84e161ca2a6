# per-kernel breakdown of the C=320 VC2 level (F=2304, 40x64) and the GEMM micro at its shapes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/level_profile.py 2304 40 64 320 3 2>&1 | tee gpurun_out/level320.log
M=$((2304*40*64))
timeout 300 python scripts/gemm_micro.py conv320=$M,320,320,3,1 qkv320=$M,960,320,1,0 o320=$M,320,320,1,1 2>&1 | tee gpurun_out/micro320.log
for bn in 160 192 256; do VINF_GEMM_BN=$bn timeout 300 python scripts/gemm_micro.py conv320=$M,320,320,3,1 o320=$M,320,320,1,1 qkv320=$M,960,320,1,0 --once 2>&1 | sed "s/^/bn=$bn /"; done
