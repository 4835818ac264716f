# NEXT-1: the paper's layouts and kernels -- parity, then the N sweep and the L x i grid.
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k paper 2>&1 | tail -3
timeout 1200 python tools/paper_sweep.py --mode n --json gpurun_out/paper_nsweep.json 2>&1 | tail -4
timeout 1800 python tools/paper_sweep.py --mode grid --reps 3 --json gpurun_out/paper_grid.json 2>&1 | tail -45
