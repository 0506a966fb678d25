#!/bin/bash
# iteration check: C3/C2 in-step timelines, a short bench line, the GPU suite, two mixed-regime points
O=gpurun_out/${1:-r02q3}; mkdir -p $O
timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 131072 > $O/c3_tl.txt 2>&1
timeout 300 python tools/timeline.py --steps 8 --batch 8 --ctx 32768 > $O/c2_tl.txt 2>&1
for f in $O/c3_tl.txt $O/c2_tl.txt; do echo "== $f"; grep -E "scan_out|verify_waited|verify_out|amend_out|complete_out" $f; done
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --full-steps 3 > $O/bench.json 2> $O/bench.err
python - $O/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).readline()); k=d['kernels']
print('step_us=%.1f'%(d['ms_per_step']*1e3), {n:(round(v['ms']*1e3,1), round(v['gbs'])) for n,v in k.items()},
      'frac=%.3f'%d['roofline']['frac'], 'e2e_us=%.1f'%(d['e2e']['ms_per_step']*1e3),
      'c2_us=%.1f'%(d['c2']['ms_per_step']*1e3 if 'c2' in d else -1), 'c2x=%.1f'%(d['c2']['speedup_vs_full_attention'] if 'c2' in d else -1))
print(json.dumps(d.get('c3mix')))
PY
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -4 $O/pytest_gpu.log
