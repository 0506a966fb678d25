#!/bin/bash
# Sweep the front (append+match) kernel variants on the C3 workload; prints step and stage times.
for v in 0 1 2 3 4 5; do
  MAC_FRONT_VARIANT=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --full-steps 3 2>/dev/null | \
  python -c "
import json,sys
d=json.loads(sys.stdin.readline())
k=d['kernels']
print('variant $v', 'step_us=%.1f'%(d['ms_per_step']*1e3), 'match_us=%.1f'%(k['mac_match']['ms']*1e3),
      'match_gbs=%.0f'%k['mac_match']['gbs'], 'amend_us=%.1f'%(k['mac_amend']['ms']*1e3),
      'complete_us=%.1f'%(k['mac_complete']['ms']*1e3), 'append_us=%.1f'%(k['mac_append_kv']['ms']*1e3))
"
done
