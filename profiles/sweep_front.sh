#!/bin/bash
# Sweep the front (append + match) kernel variants (MAC_FRONT_VARIANT) on the C3 hit-path workload.
for v in 0 1 2 3 4 5; do
  echo -n "front_variant=$v : "
  MAC_FRONT_VARIANT=$v bash profiles/quick_bench.sh --min-chunk 256 2>&1 | tail -1
done
