# Helmholtz: ncu instruction counts per precision, then bench lines (helmholtz workload, and the
# default workload to check nothing moved).
python -c "import __graft_entry__ as g; g.build()" > /dev/null
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second
for p in fp32 fp64; do
  timeout 600 ncu --kernel-name regex:p2p_tiled_helm --launch-count 2 --clock-control none --metrics $M \
    python tools/helm_bench.py --configs d16_1e6 --precisions $p --reps 1 --sample 100 > gpurun_out/helm_ncu_$p.txt 2>&1
done
python tools/helm_ipp.py fp32=gpurun_out/helm_ncu_fp32.txt fp64=gpurun_out/helm_ncu_fp64.txt
cp profiles/helm_inst_per_pair.json gpurun_out/
timeout 900 python bench.py --workload helmholtz_1e6 > gpurun_out/bench_helm.json 2> gpurun_out/bench_helm.err
timeout 900 python bench.py --workload helmholtz_1e6 --precision fp64 > gpurun_out/bench_helm64.json 2> gpurun_out/bench_helm64.err
timeout 600 python bench.py --impl reference --workload helmholtz_1e6 --steps 2 --warmup 1 > gpurun_out/bench_helm_ref.json 2>&1
tail -2 gpurun_out/bench_helm.err gpurun_out/bench_helm64.err
