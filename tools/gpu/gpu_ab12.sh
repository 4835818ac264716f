# Queue order (LPT) x tail splitting on the 1e6 density configs.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1500 python tools/sweep.py --configs d16_1e6,d32_1e6,d64_1e6 --layout tiled --tpi 2 --ns 3 --nbuf 1 --nt 128 --pad 1 --lpt 0,1 --tail 592:4,0:1,1184:4,592:8,2368:4 --reps 10
