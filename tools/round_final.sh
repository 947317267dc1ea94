#!/bin/bash
# Round-end measurements: GPU suite, smoke, bench lines for every config and the
# reference arm, ncu launch lists, full captures of the dominant kernels.
O=gpurun_out/fin; mkdir -p $O
T=/tmp/dfc_ncu; mkdir -p $T   # the .ncu-rep files stay on the box (gpurun_out is capped at 64 MiB): JSON summaries come back
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -n 3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -n 1 $O/smoke.log
for c in c5 c2 c1 c3 c4; do
  timeout 900 python bench.py --config $c > $O/bench_${c}_line.json 2> $O/bench_${c}.err
  python -c "import json;d=json.load(open('$O/bench_${c}_line.json'));print('$c', d['ms_per_step'], d['roofline']['step']['frac'], d['e2e']['value'])"
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference_line.json 2> $O/bench_ref.err; tail -c 600 $O/bench_reference_line.json
for c in c5 c2 c1 c3 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/launches_${c}.csv 2>&1
  python profiles/launch_summary.py $O/launches_${c}.csv > $O/launches_${c}_summary.txt
done
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function -k regex:"k_band_rows_fill|k_hull|k_objcol" -s 15 -c 5 -o $T/ncu_full_c5_band python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function -k regex:"k_band_summary|k_band_scan" -s 6 -c 2 -o $T/ncu_full_c5_cols python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c5_cols.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function -k regex:k_rows_anc -c 1 -o $T/ncu_full_c2_anc python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base function -k regex:k_raster_anc -c 1 -o $T/ncu_full_c4_raster python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c4.log 2>&1
for r in c5_band c5_cols c2_anc c4_raster; do
  python profiles/ncu_to_json.py $T/ncu_full_$r.ncu-rep "tools/round_final.sh (ncu --set full --import-source on --clock-control none, python bench.py --config ${r%%_*} --steps 1 --warmup 3 --no-cpu-baseline)" > $O/ncu_full_$r.json
done
python profiles/ncu_source_top.py $T/ncu_full_c5_band.ncu-rep 40 > $O/ncu_source_c5_band.txt 2>&1
