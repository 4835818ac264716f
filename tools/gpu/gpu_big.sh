# Full-size configs[3] and configs[4] on one GPU (plan build + apply).
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for W in surface_2e7 d32_7e7; do
  SECONDS=0; timeout 1200 python bench.py --workload $W --no-extras --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/big_$W.json 2> gpurun_out/big_$W.err
  echo "$W rc=$? ${SECONDS}s"; tail -2 gpurun_out/big_$W.err
done
