#!/bin/bash
# r02 iteration: C2/C3 in-step timelines (product dispatch), the GPU suite, smoke, a bench line
O=gpurun_out/${1:-r02r}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 131072 > $O/c3_tl.txt 2>&1
timeout 300 python tools/timeline.py --steps 8 --batch 8 --ctx 32768 > $O/c2_tl.txt 2>&1
for f in $O/c3_tl.txt $O/c2_tl.txt; do echo "== $f"; grep -E "verify_waited|verify_out|amend_waited|amend_out|complete_out" $f; done
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -4 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
python - $O/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).readline()); k=d['kernels']
print('step_us=%.1f'%(d['ms_per_step']*1e3), {n:(round(v['ms']*1e3,1), round(v['gbs'])) for n,v in k.items()},
      'frac=%.3f'%d['roofline']['frac'], 'full_ms=%.3f'%d['full_attention']['ms_per_step'], 'e2e_us=%.1f'%(d['e2e']['ms_per_step']*1e3),
      'hit=%.3f'%d['hit_rate'], 'c2_us=%.1f'%(d['c2']['ms_per_step']*1e3 if 'c2' in d else -1), 'c2x=%.1f'%(d['c2']['speedup_vs_full_attention'] if 'c2' in d else -1))
PY
