#!/bin/bash
# synccheck on the long-prompt tcgen05 ring build alone, then over the rest of sanitize2's set
O=gpurun_out/${1:-r02san3}; mkdir -p $O
timeout 600 python -m pytest -q -x tests/test_gpu_prefill.py::test_tcgen05_ring_build_matches_mma_at_a_long_prompt > $O/plain.log 2>&1; echo "plain rc=$?" >> $O/plain.log; tail -2 $O/plain.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_prefill.py::test_tcgen05_ring_build_matches_mma_at_a_long_prompt > $O/sync_ring.log 2>&1; echo "rc=$?" >> $O/sync_ring.log
grep -E "ERROR SUMMARY|passed|failed" $O/sync_ring.log | tail -3
T="tests/test_gpu_headline.py::test_step_graph_host_inputs_equal_pulled_inputs tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_serving.py tests/test_gpu_headline.py::test_c3_geometry_two_pass_parity"
timeout 2400 compute-sanitizer --tool synccheck --print-limit 50 python -m pytest -q -x -p no:cacheprovider $T > $O/synccheck_rest.log 2>&1; echo "rc=$?" >> $O/synccheck_rest.log
grep -E "ERROR SUMMARY|passed|failed" $O/synccheck_rest.log | tail -3
