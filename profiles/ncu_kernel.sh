#!/bin/bash
# One ncu --set full capture of the kernels matching $2 (regex) on the C3 bench.  Usage: ncu_kernel.sh <tag> <regex> [env...]
TAG=$1; RE=$2; shift 2
mkdir -p gpurun_out
env "$@" timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$RE" -s ${NCU_SKIP:-8} -c ${NCU_COUNT:-1} \
  -o gpurun_out/prof_${TAG} -f python bench.py --steps 4 --warmup 3 --no-cpu --full-steps 3 > gpurun_out/ncu_${TAG}.log 2>&1
tail -3 gpurun_out/ncu_${TAG}.log
