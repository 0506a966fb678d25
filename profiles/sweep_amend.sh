#!/bin/bash
# Sweep amend variants (MAC_AMEND_VARIANT) x min_chunk on the C3 hit-path workload.
for cfg in "0 128" "0 256" "0 64" "1 128" "3 128" "4 128" "5 128" "1 64"; do
  set -- $cfg
  echo -n "amend_variant=$1 min_chunk=$2 : "
  MAC_AMEND_VARIANT=$1 bash profiles/quick_bench.sh --min-chunk $2 2>&1 | tail -1
done
