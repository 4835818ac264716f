# compute-sanitizer over smoke (every kernel family: TILED / NR / R, device plan build, Helmholtz 2D,
# 3D, adaptive) and a slice of the new GPU tests.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san2_$tool.log 2>&1
  echo "$tool smoke rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/san2_$tool.log | tail -1
done
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q -x tests/test_device_plan.py -k "tiny" \
  tests/test_helmholtz.py -k "tiny and 1.0" > gpurun_out/san2_tests1.log 2>&1; echo "memcheck devplan/helm tests rc=$?"; tail -2 gpurun_out/san2_tests1.log
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest -q -x tests/test_3d.py -k "tiny3d or coarse" \
  tests/test_adaptive.py -k "oracle and 2000" > gpurun_out/san2_tests2.log 2>&1; echo "memcheck 3d/adaptive tests rc=$?"; tail -2 gpurun_out/san2_tests2.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest -q -x tests/test_3d.py -k "tiny3d" \
  tests/test_adaptive.py -k "oracle and 2000" > gpurun_out/san2_tests3.log 2>&1; echo "racecheck 3d/adaptive tests rc=$?"; tail -2 gpurun_out/san2_tests3.log
