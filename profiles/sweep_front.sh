#!/bin/bash
# Sweep the front (append + match) kernel variants (MAC_FRONT_VARIANT) on the C3 hit-path workload.
# 0: two-pass (128 rows/CTA, 5 CTAs/SM, default); 1: one-pass (128,5); 4: two-pass (256,4); 5: two-pass (64,8)
for v in 0 4 5 1; do
  echo -n "front_variant=$v : "
  MAC_FRONT_VARIANT=$v bash profiles/quick_bench.sh "$@" 2>&1 | tail -1
done
