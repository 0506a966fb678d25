#!/bin/bash
O=gpurun_out/${1:-r02ncutc}; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:ring_build_tc_kernel" -c 1 -o $O/prof_ring_tc -f \
  python tools/prefill_probe.py --batch 8 --ctx 32768 --reps 1 --variant tcgen05 > $O/ncu.log 2>&1
ncu -i $O/prof_ring_tc.ncu-rep --page raw --csv > $O/raw.csv 2>&1
ncu -i $O/prof_ring_tc.ncu-rep --page details --csv > $O/details.csv 2>&1
grep -o '"sm__pipe_tensor[^"]*","[^"]*","[^"]*"' $O/raw.csv | head; 
python - $O/raw.csv <<'PY'
import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr,units,vals=rows[0],rows[1],rows[2]
keys=[k for k in hdr if any(s in k for s in ("gpu__time_duration.sum","sm__pipe_tensor","sm__throughput.avg.pct","smsp__average_warp","dram__throughput.avg.pct","l1tex__data_bank_conflicts","sm__inst_executed_pipe","smsp__warp_issue_stalled","smsp__pcsamp"))]
for k in keys[:80]:
    i=hdr.index(k); print(k, vals[i], units[i])
PY
