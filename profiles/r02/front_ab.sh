#!/bin/bash
# dev library A/B on one box: two-pass scan shape (MAC_FRONT_VARIANT 0 = (512,4,16) product, 7 = (1024,4,16))
O=gpurun_out/${1:-r02front}; mkdir -p $O
DEV=$PWD/paper_2604_00235_b200/lib/libmacattn_dev.so
for rep in 1 2; do for v in ${VARS:-0 7}; do
  MACATTN_LIB=$DEV MAC_FRONT_VARIANT=$v timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu --full-steps 2 > $O/b_${v}_$rep.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/b_${v}_$rep.json').readline()); k=d['kernels']
print('variant $v', 'step %.1f scan %.1f verify %.1f c2 %.1f'%(d['ms_per_step']*1e3, k['mac_match_scan']['ms']*1e3, k['mac_match_verify']['ms']*1e3, d['c2']['ms_per_step']*1e3))"
done; done
