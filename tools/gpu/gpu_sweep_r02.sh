cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python tools/sweep.py --configs surf_2e7 --tpi 2 --ns 1,3 --nbuf 1 --nt 128,256 --tile 2,3 --reps 7 > gpurun_out/r02_sweep_surf.log 2>&1
cat gpurun_out/r02_sweep_surf.log | tail -12
timeout 900 python bench.py --precision fp64 --steps 10 --no-extras --no-cpu-baseline > gpurun_out/ab3_surf_fp64.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/ab3_surf_fp64.json').read().strip().splitlines()[-1]);print('fp64 surf', d['per_config'][0]['ms']*1e3, 'us', d['value']/1e9)"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_helmholtz.py tests/test_log_table.py -m gpu -q -x -k "fp64" 2>&1 | tail -2
