# NEXT-3 (3D): parity and bench lines.
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1200 python -m pytest tests/test_3d.py -q -m gpu 2>&1 | tail -15
for w in cube3d_1e6 cube3d_helmholtz; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  timeout 900 python bench.py --workload $w --precision fp64 --no-cpu-baseline > gpurun_out/bench_${w}_fp64.json 2> gpurun_out/bench_${w}_fp64.err
done
tail -n 3 gpurun_out/bench_cube*.err
