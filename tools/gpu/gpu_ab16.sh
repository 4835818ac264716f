# A/B: 3D box kernel CTA size (32 / 64 / 128 default / 256 threads per target box).
for v in default b3nt32 b3nt64 b3nt256; do
  if [ $v = default ]; then unset P2P_LIB; else export P2P_LIB=paper_2403_01596_b200/lib/libp2p_b200_$v.so; fi
  for w in cube3d_1e6 cube3d_helmholtz; do
    echo "== $v $w"; timeout 600 python bench.py --workload $w --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e9), round(d['roofline']['frac'],3))"
  done
done
