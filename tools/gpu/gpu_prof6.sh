# Dense TILED profiles after plan-built units + sorted items.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for C in d16_1e6 d32_1e6; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_tiled -s 3 -c 1 -o gpurun_out/p6_$C \
  python bench.py --configs $C --layout tiled --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras > /dev/null 2>&1
done
ls gpurun_out | grep p6
