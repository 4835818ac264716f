# compute-sanitizer memcheck / racecheck over smoke and a slice of the GPU parity tests.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_smoke.log 2>&1; echo "memcheck smoke rc=$?"; tail -3 gpurun_out/san_smoke.log
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "tiny or ragged or collocated or tail_split or user" > gpurun_out/san_tests.log 2>&1; echo "memcheck tests rc=$?"; tail -3 gpurun_out/san_tests.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_race.log 2>&1; echo "racecheck smoke rc=$?"; tail -3 gpurun_out/san_race.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_sync.log 2>&1; echo "synccheck smoke rc=$?"; tail -1 gpurun_out/san_sync.log
timeout 900 compute-sanitizer --tool initcheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_init.log 2>&1; echo "initcheck smoke rc=$?"; tail -1 gpurun_out/san_init.log
