#!/bin/bash
O=gpurun_out/${1:-r02san4}; mkdir -p $O
timeout 900 compute-sanitizer --tool synccheck --print-limit 5 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_prefill.py::test_tcgen05_ring_build_matches_mma_at_a_long_prompt > $O/sync_ring.log 2>&1; echo "rc=$?" >> $O/sync_ring.log
grep -E "ERROR SUMMARY|passed|failed|Barrier error" $O/sync_ring.log | sort | uniq -c | head -5
