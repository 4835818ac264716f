#!/bin/bash
# ncu --set full of the dense fp64 TILED kernel (TPI 2, lt8) on surf_2e7: pipe utilisation + source
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
T=${TAG:-f64d}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_tiled -s 3 -c 1 -o gpurun_out/${T} \
   python bench.py --precision fp64 --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras --no-e2e > gpurun_out/${T}.log 2>&1
python tools/ncu_summary.py gpurun_out/${T}.ncu-rep > gpurun_out/${T}.txt 2>&1; head -30 gpurun_out/${T}.txt
ncu -i gpurun_out/${T}.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for i,k in enumerate(h):
    if ('pipe_fp64' in k or 'pipe_alu' in k or 'pipe_fma' in k or 'pipe_xu' in k or 'pipe_lsu' in k or 'inst_executed_pipe' in k) and ('pct' in k or k.endswith('.sum')):
        print(k, v[i])
" > gpurun_out/${T}_pipes.txt; cat gpurun_out/${T}_pipes.txt | head -40
ncu -i gpurun_out/${T}.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_sass.csv 2>/dev/null
rm -f gpurun_out/${T}.ncu-rep
