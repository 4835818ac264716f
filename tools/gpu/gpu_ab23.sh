# A/B: dense span loop with 2 of every 12 logs computed on the FMA/ALU pipes (software log2, f32x2
# polynomial; libp2p_b200_swlog.so) vs all logs on MUFU (default): balancing the MUFU and FMA pipes.
python -c "import __graft_entry__ as g; g.build()" > /dev/null
P2P_LIB=paper_2403_01596_b200/lib/libp2p_b200_swlog.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "tiled and fp32" 2>&1 | tail -1
for v in default swlog default swlog; do
  if [ $v = default ]; then unset P2P_LIB; else export P2P_LIB=paper_2403_01596_b200/lib/libp2p_b200_$v.so; fi
  echo "== $v"
  timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e9), round(d['roofline']['frac'],3), [(c['config'], round(c['ms']*1e3,1)) for c in d['per_config']])"
done
