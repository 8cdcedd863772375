#!/bin/bash
# A/B of the correction passes' CG tolerance (CKKT_CG_RTOL_CORR) at C3
for r in ${RTOLS:-1e-10 1e-8 1e-6 1e-4}; do
  CKKT_CG_RTOL_CORR=$r timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rtol_$r.json 2> gpurun_out/rtol_$r.err
  python -c "
import json; d=json.load(open('gpurun_out/rtol_$r.json')); print('$r', round(d['value'],2), d['phases_ms'], d['solver'])" || tail -5 gpurun_out/rtol_$r.err
done
