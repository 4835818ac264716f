set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -5
timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -6
for W in density_1e6 lowdensity_1e7; do for L in nr tiled r; do
timeout 900 python bench.py --workload $W --layout $L --no-extras --no-cpu-baseline --steps 10 > gpurun_out/b5_${W}_$L.json 2>gpurun_out/b5_${W}_$L.err; tail -2 gpurun_out/b5_${W}_$L.err
python -c "
import json; d=json.load(open('gpurun_out/b5_${W}_$L.json'))
print('$W $L value %.4g frac %.3f' % (d['value'], d['roofline']['frac']))
for c in d['per_config']: print(c['config'], '%.1f us  %.1f Gpair/s  mufu %.3f alg %.0f GB/s k %d' % (c['ms']*1e3, c['Gpair_s'], c['frac_mufu'], c['alg_GBs'], c['tile_log2']))
"
done; done
