#!/bin/bash
# synccheck over the decode-path GPU tests (everything but the tcgen05 ring build, whose b_odone
# waits synccheck reports as "missing init", see SUMMARY)
O=gpurun_out/${1:-r02san5}; mkdir -p $O
T="tests/test_gpu_fast.py tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_diag.py tests/test_gpu_sharded.py tests/test_gpu_headline.py::test_c3_geometry_two_pass_parity tests/test_gpu_headline.py::test_adaptive_dense_mode_on_a_mixed_stream tests/test_gpu_headline.py::test_step_graph_host_inputs_equal_pulled_inputs tests/test_gpu_headline.py::test_adaptive_scan_choice_reaches_the_kernels"
timeout 3000 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest -q -p no:cacheprovider $T > $O/synccheck.log 2>&1; echo "rc=$?" >> $O/synccheck.log
grep -E "ERROR SUMMARY|passed|failed" $O/synccheck.log | tail -3
