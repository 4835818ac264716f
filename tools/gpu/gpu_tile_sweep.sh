# Tile size per dense config (the plan's rule: smallest k with >= 115 targets per non-empty tile).
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for c in d16_1e6 d32_1e6 d64_1e6; do
  for k in -1 0 1 2 3; do
    echo "== $c tile $k"; timeout 300 python bench.py --configs $c --tile $k --no-extras --no-cpu-baseline --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print([(c['config'], c['tile_log2'], round(c['ms']*1e3,1)) for c in d['per_config']])"
  done
done
