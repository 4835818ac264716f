# A/B: heavy-tile split share 1/1184 (default) vs 1/2368 and 1/4736 of the pairs (finer queue entries).
for v in default sh16 sh32 default sh16 sh32; do
  if [ $v = default ]; then unset P2P_LIB; else export P2P_LIB=paper_2403_01596_b200/lib/libp2p_b200_$v.so; fi
  echo "== $v"
  timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e9), [(c['config'], round(c['ms']*1e3,1)) for c in d['per_config']])"
  timeout 600 python bench.py --workload lowdensity_1e7 --no-extras --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e9), [(c['config'], round(c['ms']*1e3,1)) for c in d['per_config']])"
done
