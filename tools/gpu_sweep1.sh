python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1200 python tools/sweep.py --configs d16_1e6,d64_1e6,lowd1_1e7 --layout tiled --tpi 1,2 --ns 3,6 --nbuf 1,2 --tile -1 --json gpurun_out/sweep1_tiled.json
timeout 600 python tools/sweep.py --configs d16_1e6,lowd1_1e7 --layout tiled --tpi 1,2 --ns 3 --nbuf 1 --tile 1,2,3,4,5
timeout 600 python tools/sweep.py --configs d16_1e6,d64_1e6,lowd1_1e7 --layout nr --tpi 1,2 --ns 3 --nbuf 1 --tile -1
