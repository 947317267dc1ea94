#!/bin/bash
# quick C5 iteration on the GPU box: band-path parity tests, the full C5 map, bench lines
# (slice sweep), launch list.  Output under gpurun_out/quick/.
O=gpurun_out/quick; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "band or sharded or sparse or tall or tiles or point or lr_" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
tail -n 3 $O/tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c5" > $O/tests_c5.log 2>&1; echo rc=$? >> $O/tests_c5.log
tail -n 3 $O/tests_c5.log
B="python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline"
for s in ${SLICES:-1 2 4 8}; do for g in ${GROUPS_:-4}; do
  DFC_BAND_SLICES=$s DFC_BAND_GROUP=$g timeout 300 $B > $O/c5_s${s}_g$g.json 2> $O/c5_s${s}_g$g.err
  echo "slices=$s group=$g $(python -c "import json;print(json.load(open('$O/c5_s${s}_g$g.json'))['ms_per_step'])")"
done; done | tee $O/sweep.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 40 \
  python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > $O/launches.csv 2>&1
python profiles/launch_summary.py $O/launches.csv > $O/launches.txt; cat $O/launches.txt
