python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 600 python tools/sweep.py --configs lowd025_1e7,lowd1_1e7,lowd2_1e7,lowd4_1e7 --layout tiled --tpi 1 --ns 1,3 --nbuf 1 --nt 64,128 --pad 0
