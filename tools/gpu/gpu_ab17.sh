# A/B: 3D work items = 2x2x2-box tiles staging their 4x4x4 region (default) vs single boxes
# staging their 27 neighbours (P2P_TILE3D=0).
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_3d.py -q -m gpu 2>&1 | tail -2
P2P_TILE3D=0 timeout 900 python -m pytest tests/test_3d.py -q -m gpu 2>&1 | tail -1
for v in 1 0 1 0; do
  for w in cube3d_1e6 cube3d_helmholtz; do
    for p in fp32 fp64; do
      echo "== TILE3D=$v $w $p"; P2P_TILE3D=$v timeout 600 python bench.py --workload $w --precision $p --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e9), round(d['roofline']['frac'],3))"
    done
  done
done
