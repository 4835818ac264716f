# Round evidence (final code): smoke, GPU tests, bench lines, reference arm, launch list, ncu --set
# full of the step's P2P launches (density + low density) summarised on the box.
TAG=${TAG:-r01}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -3 gpurun_out/${TAG}_smoke.log
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/${TAG}_gpu_tests.log 2>&1; tail -2 gpurun_out/${TAG}_gpu_tests.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 1500 python bench.py --workload lowdensity_1e7 --steps 10 > gpurun_out/${TAG}_bench_lowd.json 2> gpurun_out/${TAG}_bench_lowd.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_ -s 9 -c 3 -o gpurun_out/${TAG}_step_full \
   python bench.py --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_ -s 12 -c 4 -o gpurun_out/${TAG}_lowd_full \
   python bench.py --workload lowdensity_1e7 --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_step_full.ncu-rep > gpurun_out/${TAG}_ncu_density_step_tiled.txt 2>&1
python tools/ncu_summary.py gpurun_out/${TAG}_lowd_full.ncu-rep > gpurun_out/${TAG}_ncu_lowdensity_step_tiled.txt 2>&1
python tools/ncu_traffic_json.py tiled_fp32 gpurun_out/${TAG}_step_full.ncu-rep d16_1e6,d32_1e6,d64_1e6 \
   gpurun_out/${TAG}_lowd_full.ncu-rep lowd025_1e7,lowd1_1e7,lowd2_1e7,lowd4_1e7 > gpurun_out/${TAG}_traffic.log 2>&1
cp profiles/ncu_summary.json gpurun_out/ncu_summary.json
rm -f gpurun_out/*.ncu-rep
ls gpurun_out | grep ${TAG}
