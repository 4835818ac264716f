# Source-level ncu capture of the dense TILED kernel on d16_1e6.
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_tiled -s 3 -c 1 -o gpurun_out/d16_full \
   python bench.py --configs d16_1e6 --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras > /dev/null 2>&1
ncu -i gpurun_out/d16_full.ncu-rep --page source --csv --print-source sass > gpurun_out/d16_sass.csv 2>/dev/null
rm -f gpurun_out/d16_full.ncu-rep
