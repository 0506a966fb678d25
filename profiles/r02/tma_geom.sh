#!/bin/bash
# dev library sweep of the TMA-fed amend's geometry (MAC_AMEND_TMA 1 = product <2,4,2>, 5-8 others)
O=gpurun_out/${1:-r02tmageom}; mkdir -p $O
DEV=$PWD/paper_2604_00235_b200/lib/libmacattn_dev.so
for rep in 1 2; do for v in 1 5 6 7 8; do
  c2=$(MACATTN_LIB=$DEV MAC_AMEND_TMA=$v timeout 300 python bench.py --workload c2 --steps 40 --warmup 5 --no-cpu --full-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step']*1e3,2))")
  m=""
  for f in 0.02 0.1; do m="$m $(MACATTN_LIB=$DEV MAC_AMEND_TMA=$v timeout 300 python tools/miss_probe.py --ctx 16384 --miss-frac $f --mode dense --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['mac_us_median'],1))")"; done
  echo "tma $v c2 $c2 mix2/10 $m"
done; done
