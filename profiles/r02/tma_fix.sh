#!/bin/bash
# TMA amend after the ring fix (NS a multiple of NC): the test that hung, 3x per variant; the C2/C3
# timelines per variant; then the full GPU suite on the product library.
O=gpurun_out/${1:-r02f}; mkdir -p $O
T=tests/test_gpu_fast.py::test_fast_long_context_hits_and_misses
for v in 1 2; do for i in 1 2 3; do
  MACATTN_LIB=$PWD/paper_2604_00235_b200/lib/libmacattn_dev.so MAC_AMEND_TMA=$v timeout 120 python -m pytest -q -x $T > $O/ab_v${v}_$i.log 2>&1; echo "tma=$v run=$i rc=$?" >> $O/ab.txt
done; done
cat $O/ab.txt
for v in 1 2 0; do
  MAC_AMEND_TMA=$v timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 131072 > $O/c3_tma$v.txt 2>&1
  MAC_AMEND_TMA=$v timeout 300 python tools/timeline.py --steps 8 --batch 8 --ctx 32768 > $O/c2_tma$v.txt 2>&1
done
for f in $O/c3_tma*.txt $O/c2_tma*.txt; do echo "== $f"; grep -E "amend_out|complete_out|amend_waited" $f; done
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -15 $O/pytest_gpu.log
