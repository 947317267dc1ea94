#!/bin/bash
# A/B of the stage-2 kernels (GPU box): DFC_ROWS=segment|win x configs.
for m in ${MODES:-segment win}; do
  for c in ${CFGS:-c2 c3 c5 c1}; do
    DFC_ROWS=$m timeout 180 python bench.py --config $c --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline > gpurun_out/ab_${c}_$m.json 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/ab_${c}_$m.json').read().strip().splitlines()[-1]); print('$m', '$c', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['step']['frac'])" 2>/dev/null || (echo "$m $c FAILED"; tail -3 gpurun_out/ab_${c}_$m.json)
  done
done
