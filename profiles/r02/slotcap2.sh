#!/bin/bash
O=gpurun_out/${1:-r02slot2}; mkdir -p $O
for rep in 1 2; do for f in 0.02 0.05 0.1 0.2; do
  timeout 300 python tools/miss_probe.py --ctx 16384 --miss-frac $f --mode dense --steps 8 >> $O/mc.jsonl 2>/dev/null
done; done
timeout 300 python tools/miss_probe.py --ctx 131072 --miss-frac 0.02 --mode dense --steps 4 >> $O/mc.jsonl 2>/dev/null
python - $O/mc.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    d=json.loads(l); print(d['ctx'], d['mode'], d['miss_frac'], d['max_chunks'], d['slot_cap'], round(d['mac_us'],1), round(d['full_us'],1))
PY
