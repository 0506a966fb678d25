#!/bin/bash
# Sweep amend variants (MAC_AMEND_VARIANT: (cp.async stages, min warps/SM) = 0: (4,7), 1: (6,4),
# 2: (2,8), 3: (3,8)) x min_chunk on C3.
for cfg in "0 128" "3 128" "3 96" "2 128" "0 96"; do
  set -- $cfg
  echo -n "amend_variant=$1 min_chunk=$2 : "
  MAC_AMEND_VARIANT=$1 bash profiles/quick_bench.sh --min-chunk $2 2>&1 | tail -1
done
