# fp64 TILED with the table log: flattened vs row loops, whole-target vs sorted row items.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for F in 1 0; do echo "== FLAT=$F"; P2P_FLAT=$F timeout 900 python tools/sweep.py --configs d16_1e6,d64_1e6,lowd1_1e7,lowd4_1e7 --layout tiled --precision fp64 --tpi 1 --ns 1 --pad 0 --nbuf 1 --nt 128 --reps 5; done
echo "== NS=3"; timeout 900 python tools/sweep.py --configs d16_1e6,d64_1e6,lowd1_1e7,lowd4_1e7 --layout tiled --precision fp64 --tpi 1 --ns 3 --pad 0 --nbuf 1 --nt 128,256 --reps 5
