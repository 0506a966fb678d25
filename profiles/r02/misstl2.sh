#!/bin/bash
# mixed regime at C3 geometry, 16K, dense mode: in-step timeline vs split-KV slots per group
O=gpurun_out/${1:-r02misstl2}; mkdir -p $O
for f in 0.02 0.1; do for mc in 8 32 64; do
  timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 16384 --miss-frac $f --mode dense --max-chunks $mc > $O/tl_${f}_${mc}.txt 2>&1
  echo "== miss $f max_chunks $mc"; grep -E "^(verify_out|dense_out|amend_in|amend_waited|amend_out|complete_waited|complete_out)" $O/tl_${f}_${mc}.txt
done; done
