#!/bin/bash
# compute-sanitizer over the round-2 code: smoke (every kernel family incl. the in-place weight
# gather, the replicated and shuffled fp64 logs) under memcheck / racecheck / synccheck /
# initcheck, and memcheck over the guard-straddle and workspace-slot tests.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_san_$tool.log 2>&1
  echo "$tool smoke rc=$?"; tail -2 gpurun_out/r02_san_$tool.log
done
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_guard_straddle.py tests/test_gpu_parity.py -q -x -k "guard or workspace or tiny" > gpurun_out/r02_san_tests.log 2>&1
echo "memcheck tests rc=$?"; tail -2 gpurun_out/r02_san_tests.log
