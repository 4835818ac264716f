# NEXT-3: Helmholtz parity, timings, and one ncu capture of the fp32 kernel (instructions per pair).
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1200 python -m pytest tests/test_helmholtz.py tests/test_device_plan.py -q -m gpu 2>&1 | tail -12
timeout 900 python tools/helm_bench.py --json gpurun_out/helm_bench.json 2>&1 | tail -8
timeout 600 ncu --kernel-name regex:p2p_tiled_helm --launch-count 2 --clock-control none \
  --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second \
  python tools/helm_bench.py --configs d16_1e6 --reps 1 --sample 100 > gpurun_out/helm_ncu.txt 2>&1
tail -40 gpurun_out/helm_ncu.txt
