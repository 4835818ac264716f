python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
export P2P_WS=0
python tools/trace.py --configs d16_1e6,d64_1e6,lowd1_1e7
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_tiled -s 3 -c 1 -o gpurun_out/t3_lowd1 python bench.py --configs lowd1_1e7 --layout tiled --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_tiled -s 3 -c 1 -o gpurun_out/t3_d16 python bench.py --configs d16_1e6 --layout tiled --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras > /dev/null 2>&1
ls gpurun_out | grep t3
