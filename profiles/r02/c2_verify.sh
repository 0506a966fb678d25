#!/bin/bash
# C2: per-head verify (product) vs per-group verify (MAC_VERIFY_PER_GROUP=1), dev library, same box
O=gpurun_out/${1:-r02c2v}; mkdir -p $O
DEV=$PWD/paper_2604_00235_b200/lib/libmacattn_dev.so
for rep in 1 2; do for k in 0 1; do
  MACATTN_LIB=$DEV MAC_VERIFY_PER_GROUP=$k timeout 600 python bench.py --workload c2 --steps 50 --warmup 5 --no-cpu --full-steps 3 > $O/c2_$k.json 2>/dev/null
  python -c "import json; d=json.loads(open('$O/c2_$k.json').readline()); print('per_group=$k', round(d['ms_per_step']*1e3,2), {n: round(v['ms']*1e3,1) for n,v in d['kernels'].items()})"
done; done
for k in 0 1; do MAC_VERIFY_PER_GROUP=$k timeout 300 python tools/timeline.py --steps 8 --batch 8 --ctx 32768 > $O/tl_$k.txt 2>&1; echo "== per_group=$k"; grep -E "^(verify_waited|verify_out|v_|amend_out|complete_out)" $O/tl_$k.txt; done
