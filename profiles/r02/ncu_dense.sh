#!/bin/bash
O=gpurun_out/${1:-r02ncudense}; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dense_kernel -c 1 -o $O/dense \
  python tools/miss_probe.py --ctx 16384 --miss-frac 0.02 --mode dense --steps 1 > $O/ncu.log 2>&1
tail -3 $O/ncu.log
