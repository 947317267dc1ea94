#!/bin/bash
# The stand-in for compute-sanitizer (closed on this GPU pool): the small
# parity cases of every kernel family with DFC_DEBUG_GUARD=1 -- canary zones
# around every scratch allocation and every output, poisoned interiors -- and a
# determinism pass (the same inputs three times, bit-identical outputs).
O=gpurun_out/guard; mkdir -p $O
DFC_DEBUG_GUARD=1 timeout ${GUARD_TIMEOUT:-1500} python -m pytest tests/test_gpu_parity.py tests/test_gpu_render.py -q -x \
  -p no:cacheprovider > $O/guard_tests.log 2>&1
echo "guard rc=$?" | tee $O/summary.txt
tail -3 $O/guard_tests.log | tee -a $O/summary.txt
timeout 600 python tools/determinism.py > $O/determinism.log 2>&1
echo "determinism rc=$?" | tee -a $O/summary.txt
tail -5 $O/determinism.log | tee -a $O/summary.txt
