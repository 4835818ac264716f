python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
export P2P_WS=0
python tools/trace.py --configs d16_1e6,d64_1e6,lowd1_1e7,surf_2e7
P2P_TPI=2 P2P_NS=3 P2P_NT=256 timeout 600 python tools/sweep.py --configs d16_1e6,d64_1e6,surf_2e7 --layout tiled --tpi 2 --ns 3 --nbuf 1 --nt 256 --pad 1
