#!/bin/bash
# compute-sanitizer over the GPU tests that cover every product kernel family: memcheck, racecheck,
# synccheck (logs -> gpurun_out/<tag>/, summaries copied to profiles/r02/)
O=gpurun_out/${1:-r02san}; mkdir -p $O
T="tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_serving.py tests/test_gpu_prefill.py::test_build_ring_gemm_form_matches_decode_steps tests/test_gpu_fast.py::test_fast_long_context_hits_and_misses tests/test_gpu_fast.py::test_step_graph_replay_equals_decode_step tests/test_gpu_headline.py::test_c3_geometry_two_pass_parity tests/test_gpu_sharded.py::test_sharded_step_matches_oracle tests/test_gpu_diag.py"
for tool in memcheck racecheck synccheck; do
  timeout 1800 compute-sanitizer --tool $tool --print-limit 50 python -m pytest -q -x -p no:cacheprovider $T > $O/$tool.log 2>&1
  echo "$tool rc=$?" >> $O/$tool.log
  tail -4 $O/$tool.log
done
