# fp64 table-driven log: parity, then fp64 TILED timings.
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | grep tiled
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 900 python tools/sweep.py --configs d16_1e6,d32_1e6,d64_1e6,lowd1_1e7,lowd4_1e7 --layout tiled --precision fp64 --tpi 1 --ns 1 --pad 0 --nbuf 1 --nt 128 --reps 5
