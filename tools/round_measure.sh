#!/bin/bash
# GPU suite + bench lines for every config + launch lists of C3/C5 (no ncu --set full).
mkdir -p gpurun_out/meas
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/meas/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/meas/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/meas/smoke.log 2>&1
for c in c2 c1 c3 c5 c4; do
  timeout 600 python bench.py --config $c > gpurun_out/meas/bench_${c}_line.json 2> gpurun_out/meas/bench_${c}.err
done
timeout 600 python bench.py --impl reference > gpurun_out/meas/bench_reference_line.json 2> gpurun_out/meas/bench_ref.err
for c in c3 c5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/meas/launches_${c}.csv 2>&1
done
