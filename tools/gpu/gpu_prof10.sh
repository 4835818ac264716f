python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_tiled -s 3 -c 1 -o gpurun_out/p10_d16_fp64 \
  python bench.py --configs d16_1e6 --layout tiled --precision fp64 --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras > /dev/null 2>&1
ls gpurun_out | grep p10
