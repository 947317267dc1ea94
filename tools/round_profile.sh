#!/bin/bash
# Round-end measurements on the GPU box: bench lines for every config, the
# reference arm, ncu launch lists and full captures of the dominant kernels.
mkdir -p gpurun_out/prof
for c in c2 c1 c3 c5 c4; do
  timeout 600 python bench.py --config $c > gpurun_out/prof/bench_${c}_line.json 2> gpurun_out/prof/bench_${c}.err
done
timeout 600 python bench.py --impl reference > gpurun_out/prof/bench_reference_line.json 2> gpurun_out/prof/bench_ref.err
for c in c2 c1 c5 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/prof/launches_${c}.csv 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function -k regex:k_rows_anc -c 2 -o gpurun_out/prof/ncu_full_c2_anc python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof/ncu_c2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function -k regex:"k_band_fill|k_band_summary|k_band_scan" -c 3 -o gpurun_out/prof/ncu_full_c5_cols python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof/ncu_c5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function -k regex:k_raster_anc -c 1 -o gpurun_out/prof/ncu_full_c4_raster python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof/ncu_c4.log 2>&1
