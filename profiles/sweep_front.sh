#!/bin/bash
# Sweep the front (append + match) kernel variants (MAC_FRONT_VARIANT) on the C3 hit-path workload.
# (ring rows per CTA, min CTAs per SM) = 0: (128,5) default, 1: (64,8), 2: (256,3)
for v in 0 1 2; do
  echo -n "front_variant=$v : "
  MAC_FRONT_VARIANT=$v bash profiles/quick_bench.sh "$@" 2>&1 | tail -1
done
