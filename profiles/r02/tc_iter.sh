#!/bin/bash
# one tcgen05-amend iteration: parity (GPU suite with every cooperative amend on it), timeline counters, bench A/B
O=gpurun_out/${1:-r02tci}; mkdir -p $O
DEV=$PWD/paper_2604_00235_b200/lib/libmacattn_dev.so
MACATTN_LIB=$DEV MAC_AMEND_TC=1 MAC_AMEND_TMA=1 timeout 900 python -m pytest tests -m gpu -q -x --timeout 200 > $O/pytest_tc.log 2>&1; echo "pytest rc=$?" >> $O/pytest_tc.log; tail -3 $O/pytest_tc.log
bash profiles/r02/tc_tl.sh $1 2>&1 | grep -v "^  .*" | head -3; grep -E "tc amend|  (softmax|producer|mma)" gpurun_out/${1:-r02tctl}/c3_tl.txt | head -6
CFGS_LIST=${CFGS_LIST:-"00 11"}
for cfg in $CFGS_LIST; do a=${cfg:0:1}; b=${cfg:1:1}
  MACATTN_LIB=$DEV MAC_AMEND_TMA=$a MAC_AMEND_TC=$b timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --full-steps 3 > $O/bench_$cfg.json 2> $O/bench_$cfg.err
  python - $O/bench_$cfg.json $cfg <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).readline())
    print('tma/tc=%s step_us=%.1f amend_us=%.1f amend_gbs=%.0f c2_us=%.1f mix2=%.1f mix10=%.1f'%(sys.argv[2], d['ms_per_step']*1e3, d['kernels']['mac_amend']['ms']*1e3, d['kernels']['mac_amend']['gbs'], d['c2']['ms_per_step']*1e3, d['c3mix']['miss_0.02']['mac_us'], d['c3mix']['miss_0.1']['mac_us']))
except Exception as e: print('bench failed', sys.argv[2], e)
PY
done
