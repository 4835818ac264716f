# ncu --set full of the P2P kernel launches of one bench step (3 densities) + the launch list.
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
TAG=${TAG:-r01}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_nr_kernel -s 3 -c 3 \
  -o gpurun_out/${TAG}_nr_full python bench.py --steps 1 --warmup 1 --profile --no-cpu-baseline --no-extras > gpurun_out/${TAG}_ncu_full.log 2>&1
tail -3 gpurun_out/${TAG}_ncu_full.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 1 --profile --no-cpu-baseline --no-extras > /dev/null 2>&1
wc -l gpurun_out/${TAG}_launches.csv
