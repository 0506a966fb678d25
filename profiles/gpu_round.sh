#!/bin/bash
# Round measurement on one B200 (run under gpurun): tests, smoke, bench (C3 default + C4),
# the C5 sweep, an ncu launch list and one ncu --set full capture of the step kernels.
# Usage: bash profiles/gpu_round.sh <tag>
TAG=${1:-r01}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
KERN='regex:front_|append_rope|match_|verify|amend_|complete_'
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k "$KERN" -c 60 --csv --log-file $O/launches.csv \
  python bench.py --steps 4 --warmup 3 --no-cpu --full-steps 3 > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "$KERN" -s 12 -c 4 \
  -o $O/prof -f python bench.py --steps 4 --warmup 3 --no-cpu --full-steps 3 > $O/ncu_full.log 2>&1
[ -n "$SKIP_SWEEP" ] || timeout 1800 python sweep.py --out $O/sweep.jsonl > $O/sweep.log 2>&1
ls -la $O
# per-launch DRAM traffic of the captured step (bench.py reads profiles/r01/ncu_traffic.json)
ncu -i $O/prof.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__registers_per_thread > $O/ncu_kernels.csv 2>/dev/null && python tools/ncu_traffic.py $O/ncu_kernels.csv > $O/ncu_traffic.json
