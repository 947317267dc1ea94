#!/bin/bash
# Rows-per-CTA sweep of the segment row pass (GPU box).
for c in ${CTAS:-256 128 512}; do
  echo "CTA=$c"; DFC_ROW_CTA=$c timeout 120 python tools/time_parts.py ${CFG:-c2} 5
done
