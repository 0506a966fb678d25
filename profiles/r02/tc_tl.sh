#!/bin/bash
O=gpurun_out/${1:-r02tctl}; mkdir -p $O
MAC_AMEND_TMA=1 MAC_AMEND_TC=1 timeout 300 python tools/timeline.py --steps 6 --batch 32 --ctx 131072 > $O/c3_tl.txt 2>&1
grep -E "^(verify_out|amend_in|amend_waited|amend_out|complete_out)|tc amend|  (softmax|producer|mma)" $O/c3_tl.txt; tail -3 $O/c3_tl.txt
