#!/bin/bash
# Profiling recipe run on the GPU box (gpurun).  Usage: bash profiles/run_profile.sh <tag> [bench args]
# 1) bench line, 2) ncu launch list of our kernels (device time + DRAM bytes),
# 3) one ncu --set full capture of each of the three step kernels.
set -x
TAG=${1:-r01}; shift
mkdir -p gpurun_out
timeout 900 python bench.py "$@" > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
KERN='regex:front_|append_rope|match_|amend_|complete_'
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k "$KERN" -c 40 --csv --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 4 --warmup 3 --no-cpu --full-steps 3 > gpurun_out/ncu_launch_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "$KERN" -s 6 -c 3 \
  -o gpurun_out/prof_${TAG} -f python bench.py --steps 4 --warmup 3 --no-cpu --full-steps 3 \
  > gpurun_out/ncu_full_${TAG}.log 2>&1
ls -la gpurun_out
