python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/dist2.json 2> gpurun_out/dist2.err; echo rc $?; tail -5 gpurun_out/dist2.err; cat gpurun_out/dist2.json | head -c 1500
