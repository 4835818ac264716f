# A/B: sparse lean path with weights read via __ldg(q + idx) in the pair loop (no per-tile gather
# phase / barrier; libp2p_b200_ldg.so) vs the shared-memory gathered copy (default).
python -c "import __graft_entry__ as g; g.build()" > /dev/null
P2P_LIB=paper_2403_01596_b200/lib/libp2p_b200_ldg.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "tiled" 2>&1 | tail -1
for v in default ldg default ldg; do
  if [ $v = default ]; then unset P2P_LIB; else export P2P_LIB=paper_2403_01596_b200/lib/libp2p_b200_$v.so; fi
  echo "== $v"
  timeout 600 python bench.py --workload lowdensity_1e7 --no-extras --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e9), round(d['roofline']['frac'],3), [(c['config'], round(c['ms']*1e3,1)) for c in d['per_config']])"
done
