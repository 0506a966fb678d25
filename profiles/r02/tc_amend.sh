#!/bin/bash
# tcgen05 amend (amend_tc.cu) through the dev library: GPU suite with every cooperative amend on it,
# then C3 / C2 bench A/B (mma / TMA / TC) and timelines
O=gpurun_out/${1:-r02tc}; mkdir -p $O
DEV=$PWD/paper_2604_00235_b200/lib/libmacattn_dev.so
MACATTN_LIB=$DEV MAC_AMEND_TC=1 MAC_AMEND_TMA=1 timeout 900 python -m pytest tests -m gpu -q -x --timeout 200 > $O/pytest_tc.log 2>&1; echo "pytest rc=$?" >> $O/pytest_tc.log; tail -5 $O/pytest_tc.log
for cfg in "0 0" "1 0" "1 1"; do set -- $cfg
  MACATTN_LIB=$DEV MAC_AMEND_TMA=$1 MAC_AMEND_TC=$2 timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --full-steps 3 > $O/bench_$1$2.json 2> $O/bench_$1$2.err
  python - $O/bench_$1$2.json $1$2 <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).readline())
    print('tma/tc=%s step_us=%.1f amend_us=%.1f amend_gbs=%.0f c2_us=%.1f'%(sys.argv[2], d['ms_per_step']*1e3, d['kernels']['mac_amend']['ms']*1e3, d['kernels']['mac_amend']['gbs'], d['c2']['ms_per_step']*1e3))
except Exception as e: print('bench failed', sys.argv[2], e)
PY
done
MAC_AMEND_TMA=1 MAC_AMEND_TC=1 timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 131072 > $O/c3_tl.txt 2>&1
MAC_AMEND_TC=1 timeout 300 python tools/timeline.py --steps 8 --batch 8 --ctx 32768 > $O/c2_tl.txt 2>&1
for f in $O/c3_tl.txt $O/c2_tl.txt; do echo "== $f"; grep -E "^(verify_out|amend_in|amend_waited|amend_out|complete_out)" $f; done
