#!/bin/bash
# Sweep the front (append + match) kernel variants (MAC_FRONT_VARIANT) on the C3 hit-path workload.
# 0: persistent tensor-core front (default); 1-3: one-shot CUDA-core stream (rows/CTA, CTAs/SM) = (128,5) (64,8) (256,3)
for v in 0 1; do
  echo -n "front_variant=$v : "
  MAC_FRONT_VARIANT=$v bash profiles/quick_bench.sh "$@" 2>&1 | tail -1
done
