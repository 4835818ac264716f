# A/B: fp32 Helmholtz series Horner chains packed in FFMA2 (default) vs scalar FFMA (helmf1).
for v in default helmf1; do
  if [ $v = default ]; then unset P2P_LIB; else export P2P_LIB=paper_2403_01596_b200/lib/libp2p_b200_$v.so; fi
  echo "== $v"; timeout 600 python tools/helm_bench.py --reps 20 --sample 2000 2>&1 | grep fp32
done
unset P2P_LIB
timeout 600 python -m pytest tests/test_helmholtz.py -q -m gpu 2>&1 | tail -2
