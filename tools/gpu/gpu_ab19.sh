# A/B: 3D fp32 Laplace with TMA-staged neighbour segments (default) vs per-source staging (P2P_BOX3_TMA=0).
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 300 python -m pytest tests/test_3d.py -q -m gpu -x 2>&1 | tail -3
for v in 1 0 1 0; do
  echo "== TMA=$v"; P2P_BOX3_TMA=$v timeout 300 python bench.py --workload cube3d_1e6 --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e9), round(d['roofline']['frac'],3), round(d['e2e']['value']/1e9))"
done
