# A/B: TILED weights gathered in-kernel through the entry index (default) vs pre-packed per
# region entry by a pack kernel and bulk-copied with the record (P2P_QPACK=1).
python -c "import __graft_entry__ as g; g.build()" > /dev/null
P2P_QPACK=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
for v in 0 1 0 1; do
  echo "== QPACK=$v"
  P2P_QPACK=$v timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e9), [(c['config'], round(c['ms']*1e3,1)) for c in d['per_config']])"
  P2P_QPACK=$v timeout 600 python bench.py --workload lowdensity_1e7 --no-extras --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e9), d['roofline']['frac'], [(c['config'], round(c['ms']*1e3,1)) for c in d['per_config']])"
done
