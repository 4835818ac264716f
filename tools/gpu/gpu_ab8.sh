# Dense tile size x CTA size sweep on the current kernel.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python tools/sweep.py --configs d16_1e6 --layout tiled --tpi 2 --ns 3 --nbuf 1 --nt 128,256 --pad 1 --tile 1,2,3 --reps 10
timeout 900 python tools/sweep.py --configs d32_1e6,d64_1e6 --layout tiled --tpi 2 --ns 3 --nbuf 1 --nt 128,256 --pad 1 --tile 0,1,2 --reps 10
