#!/bin/bash
# same-box A/B: decide_head's group counter release-only (+ acquire fence for the last head) vs acq_rel
O=gpurun_out/${1:-r02rel}; mkdir -p $O
BASE=$PWD/paper_2604_00235_b200/lib/libmacattn_base.so
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -k "two_pass or dense or adapt or c3_geometry or parity" 2>&1 | tail -1
for rep in 1 2 3; do for v in base new; do
  if [ $v = base ]; then L="MACATTN_LIB=$BASE"; else L=""; fi
  c2=$(env $L timeout 300 python bench.py --workload c2 --steps 40 --warmup 5 --no-cpu --full-steps 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step']*1e3,2))")
  m=$(env $L timeout 300 python tools/miss_probe.py --ctx 16384 --miss-frac 0.02 --mode dense --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['mac_us_median'],1))")
  echo "$v c2 $c2 mix2 $m"
done; done
