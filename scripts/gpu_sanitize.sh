# one compute-sanitizer tool per call (B200_PROFILING.md); TOOL=memcheck|synccheck|racecheck
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/sanitize_case.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool ${TOOL:-memcheck} --error-exitcode 9 python scripts/sanitize_case.py > gpurun_out/sanitize_${TOOL:-memcheck}.log 2>&1
echo "sanitizer rc=$?"; tail -8 gpurun_out/sanitize_${TOOL:-memcheck}.log
