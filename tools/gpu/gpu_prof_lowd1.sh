# Source-level ncu capture of the TILED kernel on lowd1_1e7 (the sparse roofline gap).
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_tiled -s 3 -c 1 -o gpurun_out/lowd1_full \
   python bench.py --configs lowd1_1e7 --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras > gpurun_out/lowd1_full.log 2>&1
ncu -i gpurun_out/lowd1_full.ncu-rep --page source --csv --print-source sass > gpurun_out/lowd1_sass.csv 2>/dev/null
ncu -i gpurun_out/lowd1_full.ncu-rep --page details --csv > gpurun_out/lowd1_details.csv 2>/dev/null
ls -la gpurun_out/lowd1_*
