python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
python tools/pcie_probe.py
for i in 1 2; do timeout 900 python bench.py --no-extras --no-cpu-baseline > gpurun_out/e2e_b$i.json 2>/dev/null; done
