#!/bin/bash
# mixed-regime sweep on the final build (C3 geometry, B=32): every scan mode per miss fraction, 16K and 128K
O=gpurun_out/${1:-r02msweep}; mkdir -p $O
for f in 0.0 0.01 0.02 0.05 0.1 0.2 0.3 0.5 1.0; do for mode in two_pass dense one_pass; do
  timeout 300 python tools/miss_probe.py --ctx 16384 --miss-frac $f --mode $mode --steps 10 >> $O/sweep16k.jsonl 2>/dev/null
done; done
for f in 0.0 0.02 0.1; do for mode in dense one_pass; do
  timeout 300 python tools/miss_probe.py --ctx 131072 --miss-frac $f --mode $mode --steps 4 >> $O/sweep128k.jsonl 2>/dev/null
done; done
python - $O <<'PY'
import json,sys,os
for fn in ("sweep16k.jsonl","sweep128k.jsonl"):
    rows=[json.loads(l) for l in open(os.path.join(sys.argv[1],fn))]
    print("==", fn)
    for r in rows: print(r['ctx'], r['miss_frac'], r['mode'], round(r['miss_rate'],3), round(r['mac_us_median'],1), round(r['full_us_median'],1), round(r['mac_us_median']/r['full_us_median'],3))
PY
