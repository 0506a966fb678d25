#!/bin/bash
# same-box A/B: phased piece claims in dense mode (product lib) vs lib/libmacattn_base.so
O=gpurun_out/${1:-r02phased}; mkdir -p $O
BASE=$PWD/paper_2604_00235_b200/lib/libmacattn_base.so
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -k "dense or adapt or slot or c3_geometry or graph" 2>&1 | tail -1
for rep in 1 2; do for v in base new; do
  if [ $v = base ]; then L="MACATTN_LIB=$BASE"; else L=""; fi
  m=""; for f in 0.005 0.02 0.1; do m="$m $(env $L timeout 300 python tools/miss_probe.py --ctx 16384 --miss-frac $f --mode dense --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['mac_us_median'],1))")"; done
  m128=$(env $L timeout 300 python tools/miss_probe.py --ctx 131072 --miss-frac 0.02 --mode dense --steps 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['mac_us_median'],1))")
  echo "$v 16K 0.5/2/10% $m  128K 2% $m128"
done; done
timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 16384 --miss-frac 0.02 --mode dense > $O/tl2.txt 2>&1; grep -E "^(verify_out|dense_out|amend_in|amend_waited|amend_out|complete_out)" $O/tl2.txt
