#!/bin/bash
# A/B on one box: append CTAs in the verify grid (1) vs in the scan grid (0), dev library
O=gpurun_out/${1:-r02ab}; mkdir -p $O
export MACATTN_LIB=$PWD/paper_2604_00235_b200/lib/libmacattn_dev.so
for rep in 1 2; do for k in 0 1; do
  MAC_APPEND_IN_VERIFY=$k timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu --full-steps 3 > $O/bench_${k}_${rep}.json 2>/dev/null
  python - $O/bench_${k}_${rep}.json $k <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).readline())
print('append_in_verify=%s step_us=%.2f e2e_us=%.2f c2_us=%.2f'%(sys.argv[2], d['ms_per_step']*1e3, d['e2e']['ms_per_step']*1e3, d['c2']['ms_per_step']*1e3 if 'c2' in d else -1))
PY
done; done
