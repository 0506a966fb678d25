#!/bin/bash
O=gpurun_out/${1:-r02v4}; mkdir -p $O
timeout 120 ./tools/umma_probe
timeout 600 python -m pytest -q -x tests/test_gpu_prefill.py tests/test_gpu_serving.py 2>&1 | tail -3
timeout 300 python tools/prefill_probe.py --batch 8 --ctx 32768 --reps 2 --variant tcgen05 2>&1 | tail -1
timeout 600 python tools/prefill_probe.py --batch 32 --ctx 131072 --reps 2 --variant tcgen05 2>&1 | tail -1
bash profiles/r02/e2e.sh $1
