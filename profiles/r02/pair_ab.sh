#!/bin/bash
# same-box A/B: the append's pair / 8-byte loads (product lib) vs lib/libmacattn_base.so
O=gpurun_out/${1:-r02pair}; mkdir -p $O
BASE=$PWD/paper_2604_00235_b200/lib/libmacattn_base.so
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x 2>&1 | tail -1
for rep in 1 2 3; do for v in base new; do
  if [ $v = base ]; then L="MACATTN_LIB=$BASE"; else L=""; fi
  env $L timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu --full-steps 2 > $O/b_${v}_$rep.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/b_${v}_$rep.json').readline())
print('$v', 'step %.2f e2e %.2f c2 %.2f'%(d['ms_per_step']*1e3, d['e2e']['ms_per_step']*1e3, d['c2']['ms_per_step']*1e3))"
done; done
