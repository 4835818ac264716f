python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
python tools/peaks.py > gpurun_out/peaks2.json 2>&1; cat gpurun_out/peaks2.json
export P2P_TPI=2 P2P_NS=3 P2P_NBUF=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_tiled -s 3 -c 1 -o gpurun_out/t2_d16 python bench.py --configs d16_1e6 --layout tiled --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras > /dev/null 2>&1
export P2P_TPI=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_tiled -s 3 -c 1 -o gpurun_out/t2_lowd1 python bench.py --configs lowd1_1e7 --layout tiled --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras > /dev/null 2>&1
ls gpurun_out
