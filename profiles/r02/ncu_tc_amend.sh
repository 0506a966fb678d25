#!/bin/bash
O=gpurun_out/${1:-r02ncutc}; mkdir -p $O
export MACATTN_LIB=$PWD/paper_2604_00235_b200/lib/libmacattn_dev.so MAC_AMEND_TMA=1 MAC_AMEND_TC=1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:amend_tc_kernel -s 3 -c 1 -o $O/tc_c3 \
  python bench.py --steps 2 --warmup 1 --no-cpu --full-steps 1 > $O/ncu.log 2>&1
tail -2 $O/ncu.log
