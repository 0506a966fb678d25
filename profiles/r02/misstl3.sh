#!/bin/bash
O=gpurun_out/${1:-r02misstl3}; mkdir -p $O
for f in 0.02 0.1; do
  timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 16384 --miss-frac $f --mode dense --max-chunks 32 > $O/tl_${f}.txt 2>&1
  echo "== miss $f"; grep -E "^(verify|dense|amend|complete)" $O/tl_${f}.txt
done
