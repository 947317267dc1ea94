#!/bin/bash
# quick C5 iteration on the GPU box: band-path parity tests, bench line, launch list
O=gpurun_out/quick; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "band or sharded or sparse or tall or tiles" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
timeout 300 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 40 \
  python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > $O/launches.csv 2>&1
python profiles/launch_summary.py $O/launches.csv > $O/launches.txt
