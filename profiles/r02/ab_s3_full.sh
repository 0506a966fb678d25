#!/bin/bash
# same-box A/B of the full bench line (C3 + e2e + C2 + c3mix sub-records) and the miss probes:
# _oldtree (HEAD) vs the working tree
O=gpurun_out/${1:-abs3full}; mkdir -p $O
for t in old new; do
  d=.; [ $t = old ] && d=_oldtree
  (cd $d && timeout 600 python bench.py --no-cpu --steps 30 --warmup 5 --full-steps 3 > $OLDPWD/$O/bench_$t.json 2>$OLDPWD/$O/bench_$t.err)
  for f in 0.02 0.1; do (cd $d && timeout 300 python tools/miss_probe.py --ctx 16384 --miss-frac $f --mode dense --steps 6 >> $OLDPWD/$O/miss_$t.jsonl 2>>$OLDPWD/$O/miss_$t.err); done
  (cd $d && timeout 300 python tools/miss_probe.py --ctx 4096 --miss-frac 1.0 --mode one_pass --steps 6 >> $OLDPWD/$O/miss_$t.jsonl 2>>$OLDPWD/$O/miss_$t.err)
done
python - $O <<'PY'
import json,sys
O=sys.argv[1]
for t in ("old","new"):
    try:
        d=json.loads(open(f"{O}/bench_{t}.json").readline())
        mix={k:round(v['mac_us'],1) for k,v in d.get('c3mix',{}).items() if k.startswith('miss_')}
        print(t,'c3=%.2f'%(d['ms_per_step']*1e3),'e2e=%.2f'%(d['e2e']['ms_per_step']*1e3),'c2=%.2f'%(d['c2']['ms_per_step']*1e3),'frac=%.3f'%d['roofline']['frac'],mix)
    except Exception as e: print(t,'bench failed',e)
    for l in open(f"{O}/miss_{t}.jsonl"):
        r=json.loads(l); print('  ',t,r['ctx'],r['miss_frac'],r['mode'],round(r['mac_us_median'],1),round(r['full_us_median'],1))
PY
