python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python tools/sweep.py --configs d16_1e6,d32_1e6,d64_1e6 --layout tiled --tpi 2 --ns 1,3 --nbuf 1 --nt 128,160,192,256 --pad 1
