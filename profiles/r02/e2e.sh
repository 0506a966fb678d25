#!/bin/bash
O=gpurun_out/${1:-r02e2e}; mkdir -p $O
for mode in pull host pull host; do
  if [ $mode = pull ]; then F=--e2e-pull; else F=; fi
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-sub --full-steps 3 $F > $O/bench_$mode.json 2>/dev/null
  python -c "import json; d=json.loads(open('$O/bench_$mode.json').readline()); print('$mode', 'step_us', round(d['ms_per_step']*1e3,1), 'e2e_us', round(d['e2e']['ms_per_step']*1e3,1), d['e2e'].get('max_rel_diff_vs_timed_pass_fp32'))"
done
timeout 900 python -m pytest -q -x tests/test_gpu_headline.py tests/test_gpu_fast.py 2>&1 | tail -2
