#!/bin/bash
# dev library A/B on one box: dense_kernel rows per task (MAC_DENSE_ROWS), C3 geometry at 16K, medians of 20 steps
O=gpurun_out/${1:-r02drows}; mkdir -p $O
export MACATTN_LIB=$PWD/paper_2604_00235_b200/lib/libmacattn_dev.so
for rep in 1 2; do for rows in 32 64 128; do for f in 0.02 0.1; do
  MAC_DENSE_ROWS=$rows timeout 300 python tools/miss_probe.py --ctx 16384 --miss-frac $f --mode dense --steps 20 | sed "s/^{/{\"rows\": $rows, /" >> $O/rows.jsonl 2>/dev/null
done; done; done
python - $O/rows.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    d=json.loads(l); print(d['rows'], d['miss_frac'], round(d['mac_us'],1), round(d['mac_us_median'],1), round(d['full_us_median'],1))
PY
