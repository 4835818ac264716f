#!/bin/bash
# Round-2 evidence on the final code: smoke, the whole GPU suite, bench lines (default surface_2e7
# incl. fp64 + e2e + cpu_baseline + extras; the other BASELINE workloads; the NEXT-row workloads;
# the reference arm), the ncu launch list of the default step, ncu --set full of the step's P2P
# kernel (surf_2e7) and of the sparse headline (lowd1_1e7) summarised with the source hash, and the
# 2-rank test-mode bench.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
T=${TAG:-r02}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; tail -2 gpurun_out/${T}_smoke.log
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/${T}_gpu_tests.log 2>&1; tail -2 gpurun_out/${T}_gpu_tests.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; tail -c 300 gpurun_out/${T}_bench.json
for WL in lowdensity_1e7 density_1e6; do
  timeout 900 python bench.py --workload $WL --steps 10 --no-extras > gpurun_out/${T}_bench_$WL.json 2> gpurun_out/${T}_bench_$WL.err
done
# configs[4]: "redundant vs non-redundant layout" -- the extras carry NR / R / TILED x fp32 / fp64
timeout 1800 python bench.py --workload d32_7e7 --steps 10 > gpurun_out/${T}_bench_d32_7e7.json 2> gpurun_out/${T}_bench_d32_7e7.err
for WL in helmholtz_1e6 cube3d_1e6 cube3d_helmholtz contour_2e5; do
  timeout 600 python bench.py --workload $WL --steps 10 > gpurun_out/${T}_bench_$WL.json 2> gpurun_out/${T}_bench_$WL.err
done
timeout 600 python bench.py --workload helmholtz_1e6 --precision fp64 --steps 5 > gpurun_out/${T}_bench_helmholtz_fp64.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_tiled -s 3 -c 1 -o gpurun_out/${T}_surf_full \
   python bench.py --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_tiled -s 3 -c 1 -o gpurun_out/${T}_lowd1_full \
   python bench.py --configs lowd1_1e7 --workload lowdensity_1e7 --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${T}_surf_full.ncu-rep > gpurun_out/${T}_ncu_surf.txt 2>&1
python tools/ncu_summary.py gpurun_out/${T}_lowd1_full.ncu-rep > gpurun_out/${T}_ncu_lowd1.txt 2>&1
rm -f profiles/ncu_summary.json
python tools/ncu_traffic_json.py tiled_fp32 gpurun_out/${T}_surf_full.ncu-rep surf_2e7 \
   gpurun_out/${T}_lowd1_full.ncu-rep lowd1_1e7 > gpurun_out/${T}_traffic.log 2>&1
cp profiles/ncu_summary.json gpurun_out/ncu_summary.json
# the default bench again, now with the traffic of these sources
timeout 900 python bench.py --no-extras > gpurun_out/${T}_bench_final.json 2>/dev/null
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/${T}_bench_2rank_testmode.json 2> gpurun_out/${T}_bench_2rank.err
nvidia-smi -q -d CLOCK > gpurun_out/${T}_clocks.txt 2>&1
ls gpurun_out | grep ${T}
