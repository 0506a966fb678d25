#!/bin/bash
# split-KV slots per group (max_chunks) vs the mixed regime (16K) and full attention / all-hit (128K), C3 geometry
O=gpurun_out/${1:-r02mc}; mkdir -p $O
for mc in 8 16 32 64; do
  for f in 0.02 0.1 0.3; do
    timeout 300 python tools/miss_probe.py --ctx 16384 --miss-frac $f --mode dense --max-chunks $mc --steps 6 >> $O/mc.jsonl 2>/dev/null
  done
  timeout 300 python tools/miss_probe.py --ctx 131072 --miss-frac 0.0 --mode two_pass --max-chunks $mc --steps 4 >> $O/mc.jsonl 2>/dev/null
  timeout 300 python tools/miss_probe.py --ctx 131072 --miss-frac 0.02 --mode dense --max-chunks $mc --steps 4 >> $O/mc.jsonl 2>/dev/null
done
python - $O/mc.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    d=json.loads(l); print(d['ctx'], d['mode'], d['miss_frac'], d['max_chunks'], round(d['mac_us'],1), round(d['full_us'],1))
PY
