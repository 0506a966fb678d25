#!/bin/bash
# dev library A/B on one box: dense_kernel CTAs per SM (MAC_DENSE_CTAS), C3 geometry at 16K, medians of 20 steps
O=gpurun_out/${1:-r02dgrid}; mkdir -p $O
export MACATTN_LIB=$PWD/paper_2604_00235_b200/lib/libmacattn_dev.so
for rep in 1 2; do for n in 1 2 4; do for f in 0.02 0.1; do
  MAC_DENSE_CTAS=$n timeout 300 python tools/miss_probe.py --ctx 16384 --miss-frac $f --mode dense --steps 20 | sed "s/^{/{\"ctas\": $n, /" >> $O/grid.jsonl 2>/dev/null
done; done; done
python - $O/grid.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    d=json.loads(l); print(d['ctas'], d['miss_frac'], round(d['mac_us'],1), round(d['mac_us_median'],1), round(d['full_us_median'],1))
PY
unset MACATTN_LIB
timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 16384 --miss-frac 0.02 --mode dense > $O/tl_0.02.txt 2>&1
timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 16384 --miss-frac 0.1 --mode dense > $O/tl_0.1.txt 2>&1
for f in $O/tl_0.02.txt $O/tl_0.1.txt; do echo "== $f"; grep -E "^(verify_out|dense|amend_in|amend_out|complete_out)" $f; done
