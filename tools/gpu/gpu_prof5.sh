# Dense TILED profiles (d16, d64) + sparse NT=32 A/B.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
S="--configs lowd025_1e7,lowd1_1e7,lowd2_1e7 --layout tiled --tpi 1 --ns 1 --pad 0 --reps 10 --nbuf 1"
timeout 600 python tools/sweep.py $S --nt 32,64
for C in d16_1e6 d64_1e6; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_tiled -s 3 -c 1 -o gpurun_out/p5_$C \
  python bench.py --configs $C --layout tiled --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras > /dev/null 2>&1
done
ls gpurun_out
