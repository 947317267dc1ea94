#!/bin/bash
# Tuning sweep (GPU box): row-pass segment length x config; prints value, step ms, row-pass ms.
for L in ${LS:-32 64 128}; do
  for c in ${CFGS:-c2 c3 c5}; do
    DFC_ROW_L=$L timeout 120 python bench.py --config $c --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline > gpurun_out/sw_${c}_$L.json 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/sw_${c}_$L.json').read()); print('L=$L', '$c', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['step']['frac'])" 2>/dev/null || (echo "L=$L $c FAILED"; tail -3 gpurun_out/sw_${c}_$L.json)
  done
done
