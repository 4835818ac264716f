# A/B: fp32 Helmholtz with two sources per step, the series packed in f32x2 across the sources
# (default) vs one source per step (hp0).
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_helmholtz.py tests/test_contour.py -q -m gpu 2>&1 | tail -1
for v in default hp0 default hp0; do
  if [ $v = default ]; then unset P2P_LIB; else export P2P_LIB=paper_2403_01596_b200/lib/libp2p_b200_$v.so; fi
  echo "== $v"; timeout 600 python bench.py --workload helmholtz_1e6 --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e9), [(c['config'], round(c['ms']*1e3,1)) for c in d['per_config']])"
done
