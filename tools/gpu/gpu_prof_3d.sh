python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_box3d -s 3 -c 1 -o gpurun_out/box3d_full \
   python bench.py --workload cube3d_1e6 --steps 1 --warmup 3 --profile --no-cpu-baseline > /dev/null 2>&1
ncu -i gpurun_out/box3d_full.ncu-rep --page source --csv --print-source sass > gpurun_out/box3d_sass.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/box3d_full.ncu-rep > gpurun_out/box3d_summary.txt 2>&1
rm -f gpurun_out/box3d_full.ncu-rep
