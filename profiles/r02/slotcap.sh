#!/bin/bash
# engine defaults after the span_chunks / slot_cap split (C3 geometry), then the GPU suite and a bench line
O=gpurun_out/${1:-r02slot}; mkdir -p $O
for f in 0.02 0.1 0.3; do
  timeout 300 python tools/miss_probe.py --ctx 16384 --miss-frac $f --mode dense --steps 6 >> $O/mc.jsonl 2>/dev/null
  timeout 300 python tools/miss_probe.py --ctx 16384 --miss-frac $f --mode adaptive --steps 6 >> $O/mc.jsonl 2>/dev/null
done
timeout 300 python tools/miss_probe.py --ctx 4096 --miss-frac 1.0 --mode adaptive --steps 6 >> $O/mc.jsonl 2>/dev/null
timeout 300 python tools/miss_probe.py --ctx 131072 --miss-frac 0.0 --mode two_pass --steps 4 >> $O/mc.jsonl 2>/dev/null
timeout 300 python tools/miss_probe.py --ctx 131072 --miss-frac 0.02 --mode dense --steps 4 >> $O/mc.jsonl 2>/dev/null
python - $O/mc.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    d=json.loads(l); print(d['ctx'], d['mode'], d['miss_frac'], d['max_chunks'], d['slot_cap'], round(d['mac_us'],1), round(d['full_us'],1))
PY
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -4 $O/pytest_gpu.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --full-steps 3 > $O/bench.json 2> $O/bench.err
python - $O/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).readline())
print('step_us=%.1f e2e_us=%.1f c2_us=%.1f'%(d['ms_per_step']*1e3, d['e2e']['ms_per_step']*1e3, d['c2']['ms_per_step']*1e3), json.dumps(d.get('c3mix')))
PY
