# GPU tests + bench (one JSON line) -> gpurun_out/
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -5
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
TAG=${TAG:-q}
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; tail -3 gpurun_out/bench_${TAG}.err
python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}.json'))
print('value %.4g  frac %.3f  e2e %.4g' % (d['value'], d['roofline']['frac'], d['e2e']['value'] if d.get('e2e') else 0))
for c in d['per_config']: print(c['config'], '%.1f us  %.1f Gpair/s  frac %.3f' % (c['ms']*1e3, c['Gpair_s'], c['frac_mufu']))
for c in d.get('extras', []): print(c['config'], c['layout'], c['precision'], '%.1f us %.1f Gpair/s' % (c['ms']*1e3, c['Gpair_s']))
print('cpu', d.get('cpu_baseline'))
"
if [ -n "$LOWD" ]; then
  for L in nr r; do
    timeout 900 python bench.py --workload lowdensity_1e7 --layout $L --no-extras --no-cpu-baseline --steps 10 > gpurun_out/bench_${TAG}_lowd_$L.json 2> gpurun_out/bench_${TAG}_lowd_$L.err; tail -2 gpurun_out/bench_${TAG}_lowd_$L.err
    python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}_lowd_$L.json'))
print('$L lowd value %.4g  e2e %.4g' % (d['value'], d['e2e']['value']))
for c in d['per_config']: print(c['config'], '%.1f us  %.1f Gpair/s  alg %.0f GB/s  D %.2f k %d' % (c['ms']*1e3, c['Gpair_s'], c['alg_GBs'], c['D_occ'], c['tile_log2']))
"
  done
fi
