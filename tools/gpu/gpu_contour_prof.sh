# Why is the contour Laplace step slow?  ncu of its TILED launch + per-tile trace.
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 ncu -k regex:p2p_tiled -s 3 -c 1 --clock-control none --section LaunchStats --section Occupancy --section SpeedOfLight --section WarpStateStats --section SchedulerStats \
  python bench.py --workload contour_2e5 --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras > gpurun_out/contour_ncu.txt 2>&1
grep -E "Duration|Grid Size|Block Size|Registers|Dynamic Shared|Achieved Occupancy|Theoretical Occupancy|Waves Per SM|Compute \(SM\)|Memory Throughput|Stall|Warp Cycles|Issued Warp|No Eligible|Block Limit" gpurun_out/contour_ncu.txt | head -40
python - <<'PY'
import json, torch
from paper_2403_01596_b200 import p2p, workloads as W
cfg = W.CONFIGS["contour_2e5"]
s, t, q = W.make_problem(cfg)
with p2p.Plan(s, t, level=cfg.level, layout="tiled") as pl:
    print({k: pl.info[k] for k in ("tile_log2", "tiles", "smem_bytes", "cta_threads", "slots_per_unit", "items_per_unit", "flags", "t_max", "density_occupied", "launches")})
PY
