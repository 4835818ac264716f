# fp64 table log in NR and R: parity, timings.
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | grep fp64
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for L in nr r; do timeout 900 python tools/sweep.py --configs d16_1e6,d64_1e6,lowd1_1e7 --layout $L --precision fp64 --tpi 1 --ns 1 --pad 1 --nbuf 1 --nt 128 --reps 5; done
