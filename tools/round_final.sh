#!/bin/bash
# Round-end measurements: GPU suite, smoke, bench lines for every config and the
# reference arm, ncu launch lists, full captures of the dominant kernels.
O=gpurun_out/fin; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
for c in c2 c1 c3 c5 c4; do
  timeout 600 python bench.py --config $c > $O/bench_${c}_line.json 2> $O/bench_${c}.err
done
timeout 600 python bench.py --impl reference > $O/bench_reference_line.json 2> $O/bench_ref.err
for c in c2 c1 c3 c5 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/launches_${c}.csv 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function -k regex:k_rows_anc -c 1 -o $O/ncu_full_c2_anc python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function -k regex:k_rows_lr -c 1 -o $O/ncu_full_c5_lr python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function -k regex:k_raster_anc -c 1 -o $O/ncu_full_c4_raster python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c4.log 2>&1
