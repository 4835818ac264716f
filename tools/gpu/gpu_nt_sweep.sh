# CTA size of the sparse lean TILED path (P2P_NT hook; default: 64, or 32 below 192 targets per tile).
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for nt in default 32 64 128 256; do
  if [ $nt = default ]; then unset P2P_NT; else export P2P_NT=$nt; fi
  echo "== NT=$nt"; timeout 600 python bench.py --workload lowdensity_1e7 --no-extras --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e9), round(d['roofline']['frac'],3), [(c['config'], round(c['ms']*1e3,1)) for c in d['per_config']])"
done
