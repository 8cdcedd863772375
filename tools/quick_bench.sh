#!/bin/bash
# usage: tools/quick_bench.sh "<configs>"   e.g. "c2:1072 c3:1072"
for cl in $1; do
  c=${cl%%:*}; L=${cl##*:}
  timeout 900 python bench.py --config $c --leaf $L --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_${L}.json 2> gpurun_out/bench_${c}_${L}.err
  python - <<PY
import json
try:
    d=json.load(open('gpurun_out/bench_${c}_${L}.json'))
    print('${c}:${L}', 'hykkt=%.2fms'%d['value'], 'phases', {k:round(v,2) for k,v in d['phases_ms'].items()}, 'roof', round(d['roofline']['frac'],4), d['roofline']['kernel'][:12], 'fp64', round(d['factor_fp64']['achieved_tflops'],3), 'solver', d['solver'], 'lifted', d['lifted'], 'levels', d['sizes']['n_levels'], 'ns', d['sizes']['n_supernodes'], 'launches/step', d['gpu_launches']//d['steps'], 'setup', round(d['setup_s'],1))
except Exception as e:
    print('${c}:${L} FAILED', e); print(open('gpurun_out/bench_${c}_${L}.err').read()[-2000:])
PY
done
