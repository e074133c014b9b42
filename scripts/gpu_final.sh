#!/bin/bash
# round-end measurement: benches (all configs, default flags incl. cpu_baseline / e2e), launch
# lists, and full ncu captures of each config's dominant kernel
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for c in c2 c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/final_bench_$c.json 2> gpurun_out/final_bench_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/final_bench_$c.json')); print('$c', round(d['ms_per_step'],3), d['roofline']['kernel'][:40], round(d['roofline']['frac'],3), d['clocks'])"
done
for c in c1 c2 c3 c4 c5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_$c.csv \
      python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
done
bash scripts/gpu_prof_multi.sh "c2:k_gemm_tc:1" "c4:k_gemm_tc:1" "c3:k_spa_fused:1" "c5:k_part_expand:1" "c2:k_seg_write:1"
