#!/bin/bash
# experiments: band path on C2's background plane (DFC_SPARSE_DIV), band group sweep on C5, ncu of the band path
O=gpurun_out/exp1; mkdir -p $O
for d in 8 4; do
  DFC_SPARSE_DIV=$d timeout 300 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c2_full or c1_full" > $O/c2_div$d.tests 2>&1; echo rc=$? >> $O/c2_div$d.tests
  DFC_SPARSE_DIV=$d timeout 300 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline > $O/c2_div$d.json 2> $O/c2_div$d.err
done
DFC_SPARSE_DIV=8 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 60 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > $O/launches_c2_div8.csv 2>&1
python profiles/launch_summary.py $O/launches_c2_div8.csv > $O/launches_c2_div8.txt
for g in 1 2 8 16; do
  DFC_BAND_GROUP=$g timeout 300 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline > $O/c5_g$g.json 2> $O/c5_g$g.err
done
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function \
  -k regex:"k_band_rows|k_rows_fill|k_band_hull" -s 9 -c 3 -o $O/ncu_band \
  python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_band.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function \
  -k regex:"k_band_summary|k_band_scan" -s 6 -c 2 -o $O/ncu_cols \
  python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_cols.log 2>&1
ls -la $O
