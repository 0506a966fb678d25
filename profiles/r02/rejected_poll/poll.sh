#!/bin/bash
# TMA amend claiming published items (no grid-dependency wait before the claims): suite, timelines, bench
O=gpurun_out/${1:-r02poll}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -4 $O/pytest_gpu.log
timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 16384 --miss-frac 0.02 --mode dense > $O/tl_0.02.txt 2>&1
timeout 300 python tools/timeline.py --steps 8 --batch 8 --ctx 32768 > $O/c2_tl.txt 2>&1
timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 131072 > $O/c3_tl.txt 2>&1
for f in $O/tl_0.02.txt $O/c2_tl.txt $O/c3_tl.txt; do echo "== $f"; grep -E "^(verify_out|dense_out|amend_in|amend_waited|amend_out|complete_waited|complete_out)" $f; done
for f in 0.02 0.1; do timeout 300 python tools/miss_probe.py --ctx 16384 --miss-frac $f --mode dense --steps 20 >> $O/mc.jsonl 2>/dev/null; done
timeout 300 python tools/miss_probe.py --ctx 131072 --miss-frac 0.02 --mode dense --steps 4 >> $O/mc.jsonl 2>/dev/null
python - $O/mc.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    d=json.loads(l); print(d['ctx'], d['mode'], d['miss_frac'], round(d['mac_us'],1), round(d['mac_us_median'],1), round(d['full_us_median'],1))
PY
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --full-steps 3 > $O/bench.json 2> $O/bench.err
python - $O/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).readline())
print('step_us=%.1f e2e_us=%.1f c2_us=%.1f'%(d['ms_per_step']*1e3, d['e2e']['ms_per_step']*1e3, d['c2']['ms_per_step']*1e3), json.dumps(d.get('c3mix')))
PY
