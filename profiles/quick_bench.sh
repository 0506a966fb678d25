#!/bin/bash
# Quick C3 bench summary (step time, per-stage times and GB/s, full attention, e2e).
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --full-steps 3 "$@" | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); k=d['kernels']
print('step_us=%.1f'%(d['ms_per_step']*1e3), {n:(round(v['ms']*1e3,1), round(v['gbs'])) for n,v in k.items()},
      'full_ms=%.3f'%d['full_attention']['ms_per_step'], 'speedup=%.1f'%d['speedup_vs_full_attention'],
      'e2e_us=%.1f'%(d['e2e']['ms_per_step']*1e3), 'hit=%.3f'%d['hit_rate'])
"
