# Multi-rank bench in test mode (ranks share the box's one GPU; host-staged gloo exchange):
# weak scaling (default) and strong scaling, 2 and 4 ranks.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for N in 2 4; do
  for S in weak strong; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
      bench.py --gpus $N --steps 5 --warmup 3 --scaling $S > gpurun_out/dist_${N}_${S}.json 2> gpurun_out/dist_${N}_${S}.err
    echo "N=$N $S rc=$?"; tail -c 600 gpurun_out/dist_${N}_${S}.json; tail -2 gpurun_out/dist_${N}_${S}.err
  done
done
