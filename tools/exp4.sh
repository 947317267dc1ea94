#!/bin/bash
# round-2 experiments: k_hull with searched bridges + running ORs; values-only fill with sqrt
O=gpurun_out/exp4; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "band or sharded or sparse or tall or tiles or point or lr_" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
tail -n 3 $O/tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c5" > $O/tests_c5.log 2>&1; echo rc=$? >> $O/tests_c5.log
tail -n 3 $O/tests_c5.log
B="python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline"
for g in 1 2 4 8; do for f in 4 6; do
  DFC_BAND_GROUP=$g DFC_FILL_CTAS=$f timeout 300 $B > $O/c5_g${g}_f$f.json 2> $O/c5_g${g}_f$f.err
  echo "group=$g fill_ctas=$f $(python -c "import json;print(json.load(open('$O/c5_g${g}_f$f.json'))['ms_per_step'])")"
done; done | tee $O/sweep.txt
for g in 1 4; do
DFC_BAND_GROUP=$g timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 40 \
  python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > $O/launches_g$g.csv 2>&1
python profiles/launch_summary.py $O/launches_g$g.csv > $O/launches_g$g.txt; cat $O/launches_g$g.txt
done
for d in 8; do
  DFC_SPARSE_DIV=$d timeout 300 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c2_full or c1_full" > $O/c2_div$d.tests 2>&1; echo rc=$? >> $O/c2_div$d.tests
  DFC_SPARSE_DIV=$d timeout 300 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline > $O/c2_div$d.json 2> $O/c2_div$d.err
  echo "c2 div=$d $(tail -n 1 $O/c2_div$d.tests) $(python -c "import json;print(json.load(open('$O/c2_div$d.json'))['ms_per_step'])")"
  DFC_SPARSE_DIV=$d timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 60 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > $O/launches_c2_div$d.csv 2>&1
  python profiles/launch_summary.py $O/launches_c2_div$d.csv > $O/launches_c2_div$d.txt; cat $O/launches_c2_div$d.txt
done | tee -a $O/sweep.txt
