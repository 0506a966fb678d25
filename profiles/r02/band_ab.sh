#!/bin/bash
# same-box A/B: product library (dynamic band claims) vs lib/libmacattn_base.so (static band items)
O=gpurun_out/${1:-r02band}; mkdir -p $O
BASE=$PWD/paper_2604_00235_b200/lib/libmacattn_base.so
for rep in 1 2 3; do for v in base new; do
  if [ $v = base ]; then L="MACATTN_LIB=$BASE"; else L=""; fi
  env $L timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu --full-steps 2 > $O/b_${v}_$rep.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/b_${v}_$rep.json').readline()); k=d['kernels']
print('$v', 'step %.2f amend %.1f c2 %.1f e2e %.1f mix2 %.1f'%(d['ms_per_step']*1e3, k['mac_amend']['ms']*1e3, d['c2']['ms_per_step']*1e3, d['e2e']['ms_per_step']*1e3, d['c3mix']['miss_0.02']['mac_us']))"
done; done
timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 131072 > $O/c3_tl.txt 2>&1; grep -E "^(verify_out|amend_in|amend_waited|amend_out|complete_out)" $O/c3_tl.txt
