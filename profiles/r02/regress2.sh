#!/bin/bash
# same-box C3 timelines: session-start tree vs current (slot cap default 64 / pinned 17)
O=gpurun_out/${1:-r02reg2}; mkdir -p $O
for rep in 1 2; do
  (cd _oldtree && timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 131072 > ../$O/old_$rep.txt 2>&1)
  timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 131072 > $O/new_$rep.txt 2>&1
  timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 131072 --slot-cap 17 > $O/new17_$rep.txt 2>&1
  for t in old new new17; do echo "== $t $rep"; grep -E "^(verify_waited|v_m|v_decided|verify_out|amend_waited|amend_out|complete_out)" $O/${t}_$rep.txt | tr '\n' ' '; echo; done
done
