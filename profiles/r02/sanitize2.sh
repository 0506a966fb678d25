#!/bin/bash
# compute-sanitizer memcheck + synccheck over the paths added in the second half of round 2:
# per-head verify with the KV append in its grid, dense mode with the slot-capacity split, plus
# the round's earlier product set (logs -> gpurun_out/<tag>/)
O=gpurun_out/${1:-r02san2}; mkdir -p $O
timeout 600 python -m pytest -q -x tests/test_gpu_headline.py::test_slot_capacity_spreads_missing_groups_without_changing_results > $O/new_test.log 2>&1; echo "new test rc=$?" >> $O/new_test.log; tail -3 $O/new_test.log
T="tests/test_gpu_fast.py::test_two_pass_match_large_batch_replay tests/test_gpu_headline.py::test_adaptive_dense_mode_on_a_mixed_stream tests/test_gpu_headline.py::test_slot_capacity_spreads_missing_groups_without_changing_results tests/test_gpu_headline.py::test_step_graph_host_inputs_equal_pulled_inputs tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_serving.py tests/test_gpu_headline.py::test_c3_geometry_two_pass_parity"
for tool in memcheck synccheck; do
  timeout 2400 compute-sanitizer --tool $tool --print-limit 50 python -m pytest -q -x -p no:cacheprovider $T > $O/$tool.log 2>&1
  echo "$tool rc=$?" >> $O/$tool.log
  grep -E "ERROR SUMMARY|passed|failed" $O/$tool.log | tail -3
done
