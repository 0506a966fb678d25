#!/bin/bash
# mixed-regime breakdown at C3 geometry, 16K: in-step timelines (dense mode) and the kernel launch list
O=gpurun_out/${1:-r02misstl}; mkdir -p $O
for f in 0.0 0.02 0.1; do
  timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 16384 --miss-frac $f --mode dense > $O/tl_dense_$f.txt 2>&1
done
timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 16384 --miss-frac 0.02 --mode two_pass > $O/tl_two_0.02.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__grid_size --clock-control none --csv --log-file $O/ncu_miss_0.02.csv \
  python tools/miss_probe.py --ctx 16384 --miss-frac 0.02 --mode dense --steps 3 > $O/ncu_probe.log 2>&1
for f in $O/tl_*.txt; do echo "== $f"; head -1 $f | cut -c1-200; grep -E "^(scan|verify|amend|complete|dense)" $f; grep -A3 "amend CTAs" $f | head -4; done
