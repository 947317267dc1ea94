#!/bin/bash
# C5 profile on the GPU box: plain bench line, ncu launch list, full captures
# of the band-path kernels and the column pass.  Output under gpurun_out/prof_c5/.
O=gpurun_out/prof_c5; mkdir -p $O
timeout 300 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 60 \
  python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > $O/launches.csv 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function \
  -k regex:"k_band_rows|k_rows_fill|k_hull|k_objcol" -s 18 -c 6 -o $O/ncu_band \
  python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_band.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function \
  -k regex:"k_band_summary|k_band_scan" -s 6 -c 2 -o $O/ncu_cols \
  python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_cols.log 2>&1
