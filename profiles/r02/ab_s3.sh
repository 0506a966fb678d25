#!/bin/bash
# same-box A/B: _oldtree (session-start tree) vs the working tree, C3 and C2 bench lines
# alternated, then C3 / C2 timelines of both; parity tests of the new tree
O=gpurun_out/${1:-abs3}; mkdir -p $O
for rep in 1 2 3; do
  for t in old new; do
    d=.; [ $t = old ] && d=_oldtree
    (cd $d && timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu --no-sub --full-steps 2 > $OLDPWD/$O/c3_${t}_$rep.json 2>/dev/null)
    (cd $d && timeout 300 python bench.py --workload c2 --steps 30 --warmup 5 --no-cpu --full-steps 2 > $OLDPWD/$O/c2_${t}_$rep.json 2>/dev/null)
  done
done
python - $O <<'PY'
import json,sys,glob,os
O=sys.argv[1]
for w in ("c3","c2"):
    for t in ("old","new"):
        v=[]
        for f in sorted(glob.glob(f"{O}/{w}_{t}_*.json")):
            try: d=json.loads(open(f).readline()); v.append(round(d['ms_per_step']*1e3,2))
            except Exception as e: v.append(str(e)[:40])
        print(w,t,v)
PY
for t in old new; do
  d=.; [ $t = old ] && d=_oldtree
  (cd $d && timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 131072 > $OLDPWD/$O/tl_c3_$t.txt 2>&1)
  (cd $d && timeout 300 python tools/timeline.py --steps 8 --batch 8 --ctx 32768 > $OLDPWD/$O/tl_c2_$t.txt 2>&1)
  for w in c3 c2; do echo "== $w $t"; grep -E "^(verify_out|amend_waited|amend_out|complete_out)" $O/tl_${w}_$t.txt | tr -s ' ' | tr '\n' '|'; echo; done
done
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; tail -2 $O/pytest.log
