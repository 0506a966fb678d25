#!/bin/bash
# dev library A/B on one box: the mma amend's K/V loads L2 evict-first (default) vs normal priority
# (MAC_AMEND_VARIANT=4: the hit kernel without the hint); step, full attention, complete's DRAM bytes
O=gpurun_out/${1:-r02evict}; mkdir -p $O
DEV=$PWD/paper_2604_00235_b200/lib/libmacattn_dev.so
for rep in 1 2; do for v in def 4; do
  if [ $v = def ]; then VAR=""; else VAR="MAC_AMEND_VARIANT=$v"; fi
  env MACATTN_LIB=$DEV $VAR timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu --full-steps 3 --no-sub > $O/b_${v}_$rep.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/b_${v}_$rep.json').readline()); k=d['kernels']
print('amend $v', 'step %.2f amend %.1f complete %.1f full_ms %.3f e2e %.1f'%(d['ms_per_step']*1e3, k['mac_amend']['ms']*1e3, k['mac_complete']['ms']*1e3, d['full_attention']['ms_per_step'], d['e2e']['ms_per_step']*1e3))"
done; done
for v in def 4; do
  if [ $v = def ]; then VAR=""; else VAR="MAC_AMEND_VARIANT=$v"; fi
  env MACATTN_LIB=$DEV $VAR timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none \
    -k "regex:complete_bf16|amend_mma" -s 6 -c 4 --csv python bench.py --steps 4 --warmup 3 --no-cpu --no-sub --full-steps 1 > $O/ncu_$v.csv 2>/dev/null
  echo "== ncu $v"; grep -E "complete_bf16|amend_mma" $O/ncu_$v.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-160 | head -8
done
