#!/bin/bash
# same-box A/B: the session-start tree (e8fd5b5, built into _oldtree/) vs the current tree, C3 bench
O=gpurun_out/${1:-r02reg}; mkdir -p $O
for rep in 1 2 3; do
  (cd _oldtree && timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu --full-steps 2 --no-sub > ../$O/old_$rep.json 2>/dev/null)
  timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu --full-steps 2 --no-sub > $O/new_$rep.json 2>/dev/null
  for t in old new; do python -c "
import json; d=json.loads(open('$O/${t}_$rep.json').readline()); k=d['kernels']
print('$t', 'step %.1f  scan %.1f verify %.1f amend %.1f complete %.1f'%(d['ms_per_step']*1e3, k['mac_match_scan']['ms']*1e3, k['mac_match_verify']['ms']*1e3, k['mac_amend']['ms']*1e3, k['mac_complete']['ms']*1e3))"; done
done
