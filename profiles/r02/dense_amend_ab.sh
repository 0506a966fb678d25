#!/bin/bash
# dense mode (match_mode 2): TMA-fed amend (product) vs the one-warp amend (MAC_AMEND_TMA=0), dev library
O=gpurun_out/${1:-r02damend}; mkdir -p $O
DEV=$PWD/paper_2604_00235_b200/lib/libmacattn_dev.so
for rep in 1 2; do for f in 0.0 0.005 0.02 0.1 0.2; do for t in d 0; do
  if [ $t = d ]; then E=""; else E="MAC_AMEND_TMA=0"; fi
  env MACATTN_LIB=$DEV $E timeout 300 python tools/miss_probe.py --ctx 16384 --miss-frac $f --mode dense --steps 10 | sed "s/^{/{\"tma\": \"$t\", /" >> $O/ab.jsonl 2>/dev/null
done; done; done
for t in d 0; do if [ $t = d ]; then E=""; else E="MAC_AMEND_TMA=0"; fi
  env MACATTN_LIB=$DEV $E timeout 300 python tools/miss_probe.py --ctx 131072 --miss-frac 0.02 --mode dense --steps 4 | sed "s/^{/{\"tma\": \"$t\", /" >> $O/ab.jsonl 2>/dev/null; done
python - $O/ab.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    d=json.loads(l); print(d['tma'], d['ctx'], d['miss_frac'], round(d['mac_us_median'],1))
PY
