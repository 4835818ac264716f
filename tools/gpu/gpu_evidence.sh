# Round evidence: GPU tests, default bench line, low-density bench, ncu launch list and a full capture
# of the P2P kernels of one bench step.  Outputs under gpurun_out/ (copy summaries to profiles/).
set -x
TAG=${TAG:-r01}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -7
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -4
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -2 gpurun_out/${TAG}_bench.err
timeout 1500 python bench.py --workload lowdensity_1e7 --steps 10 > gpurun_out/${TAG}_bench_lowd.json 2> gpurun_out/${TAG}_bench_lowd.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_ -s 9 -c 3 -o gpurun_out/${TAG}_step_full \
   python bench.py --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_ -s 12 -c 4 -o gpurun_out/${TAG}_lowd_full \
   python bench.py --workload lowdensity_1e7 --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras > /dev/null 2>&1
ls gpurun_out | grep ${TAG}
