python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
P2P_TPI=4 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tiled and fp32" 2>&1 | tail -2
timeout 900 python tools/sweep.py --configs d16_1e6,d32_1e6,d64_1e6,surf_2e7 --layout tiled --tpi 4,2 --ns 3,1 --nbuf 1 --nt 64,128 --pad 1
