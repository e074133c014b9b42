#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for c in c2 c2b c3; do
  timeout 600 python bench.py --config $c --also "" --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
  python -c "import json; d=json.load(open('gpurun_out/b_$c.json')); print('$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, d['config']['path'], d['roofline']['frac'], d['selector_calibration'])" || tail -3 gpurun_out/b_$c.err
done
for c in c5 c4s; do
  TCUDB_CALIBRATE=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --also "" --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
  echo "== $c"; python scripts/launch_table.py gpurun_out/launches_$c.csv 14
done
bash scripts/gpu_prof_multi.sh "c5:k_part_scatter:1" "c5:k_part_hist:1" "c5:k_part_expand:1" "c5:k_hash_insert_smem:1" "c5:k_col_stats:1" "c5:k_group_codes:1"
python scripts/ncu_summary.py "c5 kernels, round 2" gpurun_out/r02_c5_ncu.txt gpurun_out/prof_c5_*.ncu-rep
