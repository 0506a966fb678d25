#!/bin/bash
# A/B the TMA amend on the test that hung / crashed: dev library (MAC_DEV_KNOBS) so MAC_AMEND_TMA
# can switch the hit amend back to the one-warp mma kernel; then sanitizers on the TMA path.
O=gpurun_out/${1:-r02t}; mkdir -p $O
export MACATTN_LIB=$PWD/paper_2604_00235_b200/lib/libmacattn_dev.so
T=tests/test_gpu_fast.py::test_fast_long_context_hits_and_misses
for tma in 0 1; do for i in 1 2 3; do
  MAC_AMEND_TMA=$tma timeout 120 python -m pytest -q -x $T > $O/ab_tma${tma}_$i.log 2>&1; echo "tma=$tma run=$i rc=$?" >> $O/ab.txt
done; done
cat $O/ab.txt
timeout 300 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest -q -x $T > $O/synccheck.log 2>&1; echo "synccheck rc=$?" >> $O/synccheck.log; tail -4 $O/synccheck.log
timeout 300 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest -q -x $T > $O/racecheck.log 2>&1; echo "racecheck rc=$?" >> $O/racecheck.log; tail -4 $O/racecheck.log
MAC_AMEND_TMA=0 timeout 900 python -m pytest -q tests/test_gpu_api.py tests/test_gpu_serving.py tests/test_gpu_prefill.py tests/test_gpu_fast.py tests/test_gpu_headline.py "tests/test_gpu_sharded.py::test_nccl_kv_sharded_step_across_visible_gpus" > $O/newtests.log 2>&1; echo "newtests rc=$?" >> $O/newtests.log; tail -30 $O/newtests.log
