#!/bin/bash
# r02 final measurement: GPU suite, smoke, bench line, the ncu launch list of the bench command,
# one ncu --set full capture of the dominant kernel (C3 amend), the C2 TMA amend, the dense kernel
# (mixed step) and the ring build; timelines of C2 / C3; prefill probe.
O=gpurun_out/${1:-r02final}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
KERN='regex:front_|append_|match_|verify_|dense_|amend_|complete_'
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k "$KERN" -c 60 --csv --log-file $O/launches_c3.csv python bench.py --steps 4 --warmup 3 --no-cpu --no-sub --full-steps 3 > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:amend_mma_kernel|front_half_kernel|verify_kernel|complete_bf16" -s 8 -c 4 \
  -o $O/prof_c3 -f python bench.py --steps 4 --warmup 3 --no-cpu --no-sub --full-steps 3 > $O/ncu_full_c3.log 2>&1
ncu -i $O/prof_c3.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__occupancy_limit_registers > $O/ncu_kernels_c3.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:amend_tma_kernel" -s 2 -c 1 \
  -o $O/prof_c2_tma -f python bench.py --workload c2 --steps 3 --warmup 3 --no-cpu --full-steps 2 > $O/ncu_full_c2.log 2>&1
ncu -i $O/prof_c2_tma.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed > $O/ncu_kernels_c2_tma.csv 2>&1
timeout 600 ncu --set full --clock-control none -k "regex:ring_build_tc_kernel" -c 1 -o $O/prof_ring -f \
  python tools/prefill_probe.py --batch 8 --ctx 32768 --reps 1 --variant tcgen05 > $O/ncu_ring.log 2>&1
ncu -i $O/prof_ring.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread > $O/ncu_ring.csv 2>&1
for v in tcgen05 mma; do timeout 600 python tools/prefill_probe.py --batch 32 --ctx 131072 --reps 2 --variant $v >> $O/prefill.jsonl 2>>$O/prefill.err; done
timeout 300 python tools/prefill_probe.py --batch 8 --ctx 32768 --reps 2 --variant tcgen05 >> $O/prefill.jsonl 2>>$O/prefill.err
cat $O/prefill.jsonl
timeout 300 python tools/timeline.py --steps 8 --batch 32 --ctx 131072 > $O/c3_tl.txt 2>&1
timeout 300 python tools/timeline.py --steps 8 --batch 8 --ctx 32768 > $O/c2_tl.txt 2>&1
for f in $O/c3_tl.txt $O/c2_tl.txt; do echo "== $f"; grep -E "scan_out|verify_waited|verify_out|amend_out|complete_out" $f; done
for f in 0.02 0.1; do timeout 300 python tools/miss_probe.py --ctx 16384 --miss-frac $f --mode dense --steps 6 >> $O/miss.jsonl 2>>$O/miss.err; done
timeout 300 python tools/miss_probe.py --ctx 4096 --miss-frac 1.0 --mode one_pass --steps 6 >> $O/miss.jsonl 2>>$O/miss.err
cat $O/miss.jsonl
python - $O/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).readline()); k=d['kernels']
print('step_us=%.1f'%(d['ms_per_step']*1e3), {n:(round(v['ms']*1e3,1), round(v['gbs'])) for n,v in k.items()},
      'frac=%.3f'%d['roofline']['frac'], 'full_ms=%.3f'%d['full_attention']['ms_per_step'], 'e2e_us=%.1f'%(d['e2e']['ms_per_step']*1e3),
      'c2_us=%.1f'%(d['c2']['ms_per_step']*1e3 if 'c2' in d else -1), 'c2x=%.1f'%(d['c2']['speedup_vs_full_attention'] if 'c2' in d else -1))
print(json.dumps(d.get('c3mix')))
PY
head -c 600 $O/bench_reference.json
cuobjdump -sass paper_2604_00235_b200/lib/libmacattn.so | grep -oE "UTCHMMA|UTMALDG|LDTM|STTM|UTCBAR|HMMA\.16816[^ ]*|SYNCS[^ ]*" | sort | uniq -c > $O/sass_mnemonics.txt 2>&1
