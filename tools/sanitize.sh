#!/bin/bash
# compute-sanitizer over the small parity cases of every kernel family
# (SURVEY.md section 5).  Output: gpurun_out/sanitize/<tool>.log + summary.txt
O=gpurun_out/sanitize; mkdir -p $O
SEL="six_point or polarity_inside or dual_polarity or batched_points or band_sparse_random or band_sparse_full_row or band_sparse_ties or band_sparse_inverted or point_planes or point_plane_dual or raster_random or lr_row_kernel or lr_overflow or anc_row_kernel or anc_ties or merge_row_kernel or dense_rows or sharded_library_in_process or raster_pass or row_owners or vertical or band_scan_medium or envelope_from or label_ordinals or column_striped"
: > $O/summary.txt
for tool in memcheck racecheck initcheck synccheck; do
  extra=""
  [ $tool = initcheck ] && extra="--track-unused-memory no"
  timeout ${SAN_TIMEOUT:-1500} compute-sanitizer --tool $tool $extra --target-processes all --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_render.py -q -x -p no:cacheprovider -k "$SEL" > $O/$tool.log 2>&1
  echo "$tool rc=$?" >> $O/summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" $O/$tool.log | tail -4 >> $O/summary.txt
done
cat $O/summary.txt
