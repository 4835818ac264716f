# A/B: 3D staging by warp per neighbour segment (default) vs per-source segment search (ws0).
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_3d.py -q -m gpu 2>&1 | tail -1
for v in default ws0 default ws0; do
  if [ $v = default ]; then unset P2P_LIB; else export P2P_LIB=paper_2403_01596_b200/lib/libp2p_b200_$v.so; fi
  for w in cube3d_1e6 cube3d_helmholtz; do
    echo "== $v $w"; timeout 600 python bench.py --workload $w --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e9), round(d['roofline']['frac'],3))"
  done
done
