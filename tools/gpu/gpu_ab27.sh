# A/B: 3D Helmholtz fp32 with two targets per thread (default) vs one (bh0).
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_3d.py -q -m gpu 2>&1 | tail -1
for v in default bh0 default bh0; do
  if [ $v = default ]; then unset P2P_LIB; else export P2P_LIB=paper_2403_01596_b200/lib/libp2p_b200_$v.so; fi
  echo "== $v"; timeout 600 python bench.py --workload cube3d_helmholtz --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e9), round(d['roofline']['frac'],3))"
done
