# ncu --set full with source of the sparse TILED kernel (lean path, defaults) on lowd1 and lowd025.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for C in lowd1_1e7 lowd025_1e7; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_tiled -s 3 -c 1 -o gpurun_out/p4_$C \
  python bench.py --configs $C --layout tiled --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras > /dev/null 2>&1
done
ls gpurun_out
