python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tiled" 2>&1 | tail -2
timeout 600 python tools/sweep.py --configs d16_1e6,d32_1e6,d64_1e6 --layout tiled --tpi 2 --ns 3 --nbuf 1 --nt 128 --pad 1
timeout 600 python tools/sweep.py --configs lowd025_1e7,lowd1_1e7,lowd2_1e7,lowd4_1e7 --layout tiled --tpi 1 --ns 1 --nbuf 1 --nt 64,128,256 --pad 0
