python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
export P2P_WS=0
timeout 1200 python tools/sweep.py --configs d16_1e6 --layout tiled --tpi 2 --ns 3 --nbuf 1 --nt 32,64,128 --pad 1 --tile 1,2
timeout 1200 python tools/sweep.py --configs d32_1e6 --layout tiled --tpi 2 --ns 3 --nbuf 1 --nt 32,64,128 --pad 1 --tile 0,1,2
timeout 1200 python tools/sweep.py --configs d64_1e6 --layout tiled --tpi 2 --ns 3 --nbuf 1 --nt 32,64,128 --pad 1 --tile 0,1
timeout 1200 python tools/sweep.py --configs lowd1_1e7 --layout tiled --tpi 1 --ns 1 --nbuf 1 --nt 32,64,128 --pad 0 --tile 3,4
timeout 1200 python tools/sweep.py --configs lowd025_1e7 --layout tiled --tpi 1 --ns 1 --nbuf 1 --nt 32,64,128 --pad 0 --tile 4,5
