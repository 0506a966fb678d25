#!/bin/bash
# memcheck one GPU test (arg 2: -k expression), then the whole GPU suite without -x
O=gpurun_out/${1:-r02d}; K=${2:-test_fast_long_context_hits_and_misses}
mkdir -p $O
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests -m gpu -q -x -k "$K" > $O/memcheck.log 2>&1; echo "memcheck rc=$?" >> $O/memcheck.log
tail -5 $O/memcheck.log
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -15 $O/pytest_gpu.log
