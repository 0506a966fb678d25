#!/bin/bash
# quick iteration on one B200: the GPU suite (or a -k subset), then a short C3 bench line summary
O=gpurun_out/${1:-r02q}; K=${2:-}
mkdir -p $O
if [ -n "$K" ]; then timeout 900 python -m pytest tests -m gpu -q -x -k "$K" > $O/pytest_gpu.log 2>&1
else timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; fi
echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -3 $O/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --full-steps 3 > $O/bench.json 2> $O/bench.err
python - $O/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).readline()); k=d['kernels']
print('step_us=%.1f'%(d['ms_per_step']*1e3), {n:(round(v['ms']*1e3,1), round(v['gbs'])) for n,v in k.items()},
      'frac=%.3f'%d['roofline']['frac'], 'full_ms=%.3f'%d['full_attention']['ms_per_step'], 'e2e_us=%.1f'%(d['e2e']['ms_per_step']*1e3),
      'hit=%.3f'%d['hit_rate'], 'c2_us=%.1f'%(d['c2']['ms_per_step']*1e3 if 'c2' in d else -1), 'c2x=%.1f'%(d['c2']['speedup_vs_full_attention'] if 'c2' in d else -1))
PY
