#!/bin/bash
# miss / mixed regime at C3 geometry: MAC step vs full attention per scan mode; then the GPU suite
O=gpurun_out/${1:-r02m}; mkdir -p $O
for ctx in 4096 16384; do
  for f in 0.02 0.1 0.3 1.0; do
    for mode in dense one_pass adaptive; do
      timeout 300 python tools/miss_probe.py --ctx $ctx --miss-frac $f --mode $mode --steps 8 >> $O/miss.jsonl 2>> $O/miss.err
    done
  done
done
timeout 300 python tools/miss_probe.py --ctx 16384 --miss-frac 0.02 --mode two_pass --steps 8 >> $O/miss.jsonl 2>> $O/miss.err
cat $O/miss.jsonl
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -6 $O/pytest_gpu.log
timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 131072 > $O/c3_tl.txt 2>&1
timeout 300 python tools/timeline.py --steps 8 --batch 8 --ctx 32768 > $O/c2_tl.txt 2>&1
for f in $O/c3_tl.txt $O/c2_tl.txt; do echo "== $f"; grep -E "scan_out|verify_waited|verify_out|amend_out|complete_out" $f; done
