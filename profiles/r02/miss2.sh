#!/bin/bash
# mixed regime: split-KV slots per group and the TMA amend (dev library) vs the miss path's long items
O=gpurun_out/${1:-r02m2}; mkdir -p $O
run() { timeout 300 python tools/miss_probe.py --steps 6 "$@" >> $O/miss.jsonl 2>> $O/miss.err; }
for mc in 8 32 96; do
  run --ctx 16384 --miss-frac 0.02 --mode dense --max-chunks $mc
  run --ctx 16384 --miss-frac 0.1 --mode dense --max-chunks $mc
  run --ctx 16384 --miss-frac 0.02 --mode one_pass --max-chunks $mc
  run --ctx 4096 --miss-frac 1.0 --mode one_pass --max-chunks $mc
done
export MACATTN_LIB=$PWD/paper_2604_00235_b200/lib/libmacattn_dev.so
for mc in 8 32; do
  MAC_AMEND_TMA=1 run --ctx 16384 --miss-frac 0.02 --mode dense --max-chunks $mc
  MAC_AMEND_TMA=1 run --ctx 16384 --miss-frac 0.1 --mode dense --max-chunks $mc
  MAC_AMEND_TMA=1 run --ctx 4096 --miss-frac 1.0 --mode one_pass --max-chunks $mc
done
unset MACATTN_LIB
for mc in 17 64 128; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-sub --full-steps 5 --max-chunks $mc > $O/bench_mc$mc.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('$O/bench_mc$mc.json').readline()); print('max_chunks $mc', 'mac_us', round(d['ms_per_step']*1e3,1), 'full_ms', d['full_attention']['ms_per_step'])"
done
cat $O/miss.jsonl
timeout 900 python tools/prefill_probe.py --batch 32 --ctx 131072 --reps 2 > $O/prefill_c3.json 2>&1; cat $O/prefill_c3.json | tail -3
timeout 300 python tools/prefill_probe.py --batch 8 --ctx 32768 --reps 2 > $O/prefill_c2.json 2>&1; cat $O/prefill_c2.json | tail -3
