#!/bin/bash
# A/B of two builds on the same box: lib_ab/libdfc_$A.so vs lib_ab/libdfc_$B.so, alternating.
# usage: tools/ab.sh A B "cfg chunks" ...
A=$1; B=$2; shift 2
for rep in 1 2; do
  for v in $A $B; do
    for c in "$@"; do
      DFC_LIB=paper_2106_03503_b200/lib_ab/libdfc_$v.so timeout 300 python tools/lr_sweep.py $c 0 2>&1 | grep default | sed "s/^/$v /"
    done
  done
done
