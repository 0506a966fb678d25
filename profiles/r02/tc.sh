#!/bin/bash
O=gpurun_out/${1:-r02tc}; mkdir -p $O
timeout 600 python -m pytest -q -x tests/test_gpu_prefill.py > $O/prefill_tests.log 2>&1; echo "rc=$?" >> $O/prefill_tests.log; tail -15 $O/prefill_tests.log
for v in tcgen05 mma; do timeout 300 python tools/prefill_probe.py --batch 8 --ctx 32768 --reps 2 --variant $v 2>&1 | tail -1; done
timeout 600 python tools/prefill_probe.py --batch 32 --ctx 131072 --reps 2 --variant tcgen05 2>&1 | tail -1
