#!/bin/bash
# in-step kernel timelines (MAC_TIMELINE + dev-knob build): C3 and C2, TMA amend on / off
O=gpurun_out/${1:-r02tl}; mkdir -p $O
for tma in 1 0; do
  MAC_AMEND_TMA=$tma timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 131072 > $O/c3_tma$tma.txt 2>&1
  MAC_AMEND_TMA=$tma timeout 300 python tools/timeline.py --steps 8 --batch 8 --ctx 32768 > $O/c2_tma$tma.txt 2>&1
done
for f in $O/c3_tma1.txt $O/c3_tma0.txt $O/c2_tma1.txt $O/c2_tma0.txt; do echo "== $f"; grep -v "^{" $f | head -14; done
