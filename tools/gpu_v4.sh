set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -5
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
for W in density_1e6 lowdensity_1e7; do for L in nr r; do
timeout 900 python bench.py --workload $W --layout $L --no-extras --no-cpu-baseline --steps 10 > gpurun_out/b4_${W}_$L.json 2>gpurun_out/b4_${W}_$L.err; tail -2 gpurun_out/b4_${W}_$L.err
python -c "
import json; d=json.load(open('gpurun_out/b4_${W}_$L.json'))
print('$W $L value %.4g frac %.3f' % (d['value'], d['roofline']['frac']))
for c in d['per_config']: print(c['config'], '%.1f us  %.1f Gpair/s  mufu %.3f alg %.0f GB/s k %d' % (c['ms']*1e3, c['Gpair_s'], c['frac_mufu'], c['alg_GBs'], c['tile_log2']))
"
done; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_nr_kernel -s 3 -c 1 -o gpurun_out/v4_d16 python bench.py --configs d16_1e6 --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_nr_kernel -s 3 -c 1 -o gpurun_out/v4_lowd1 python bench.py --configs lowd1_1e7 --steps 1 --warmup 3 --profile --no-cpu-baseline --no-extras > /dev/null 2>&1
ls -la gpurun_out/
