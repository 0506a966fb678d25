#!/bin/bash
# L2 prefetch of the hit step's certain K/V: sweep the piece tokens prefetched per group
O=gpurun_out/${1:-r02pf}; mkdir -p $O
for pf in 0 256 512 128; do
  MAC_PREFETCH_TOKENS=$pf timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 131072 > $O/c3_tl_pf$pf.txt 2>&1
  MAC_PREFETCH_TOKENS=$pf timeout 300 python tools/timeline.py --steps 8 --batch 8 --ctx 32768 > $O/c2_tl_pf$pf.txt 2>&1
  echo "== pf=$pf"; grep -E "amend_out|complete_out" $O/c3_tl_pf$pf.txt $O/c2_tl_pf$pf.txt
done
export MACATTN_LIB=$PWD/paper_2604_00235_b200/lib/libmacattn_dev.so
for pf in 0 256 512; do
  MAC_PREFETCH_TOKENS=$pf timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-sub --full-steps 3 > $O/bench_pf$pf.json 2>/dev/null
  python -c "import json; d=json.loads(open('$O/bench_pf$pf.json').readline()); print('pf $pf step_us', round(d['ms_per_step']*1e3,1), {n:round(v['ms']*1e3,1) for n,v in d['kernels'].items()})"
done
