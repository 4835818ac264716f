python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 ncu -k regex:p2p_box3d -s 3 -c 1 --clock-control none --import-source on --section SpeedOfLight --section WarpStateStats --section SourceCounters --section InstructionStats --section Occupancy \
  --metrics smsp__thread_inst_executed.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__average_warp_latency_issue_stalled_barrier.ratio,smsp__pcsamp_warps_issue_stalled_barrier,lts__t_bytes.sum \
  python bench.py --workload cube3d_1e6 --steps 1 --warmup 3 --profile --no-cpu-baseline > gpurun_out/3d_ncu.txt 2>&1
sed -n '/box3d/,$p' gpurun_out/3d_ncu.txt | grep -v "^\s*$" | head -150
