#!/bin/bash
# round-2 evidence: default bench (all configs), launch lists and ncu captures per config
# (calibration constants of the bench run injected), GPU tests, 300-seed fuzz, selector sweep,
# compute-sanitizer. Every step under a hard-kill timeout.
set -u
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
export TAG=${TAG:-r02}
( time timeout -s KILL 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err ) 2> gpurun_out/${TAG}_bench.time
tail -3 gpurun_out/${TAG}_bench.time
export TCUDB_CALIBRATION_VALUES=$(python -c "
import json; c=json.load(open('gpurun_out/${TAG}_bench.json'))['selector_calibration']
print(','.join(repr(c[k]) for k in ('R_i8','R_bf16','R_fp4','BW','R_sp','T_sp0','T_d0')))")
echo "calibration: $TCUDB_CALIBRATION_VALUES"
python - <<'PY'
import json, os
d=json.load(open('gpurun_out/'+os.environ['TAG']+'_bench.json'))
print('c2', round(d['ms_per_step'],3), d['roofline']['frac'], d['query_roofline']['frac'], d['clocks'])
for c,r in d['configs'].items():
    print(c, round(r['ms_per_step'],3), r['config']['path'], round(r['roofline']['frac'],3), r['query_roofline']['frac'])
PY
for c in c1 c2 c3 c4 c5 c2b c4s; do
  timeout -s KILL 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/${TAG}_launches_$c.csv \
      python bench.py --config $c --also "" --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
done
rm -f gpurun_out/prof_*.ncu-rep
bash scripts/gpu_prof_multi.sh "c2:k_gemm_tc:1" "c4:k_gemm_tc:1" "c3:k_spa_fused:1" "c5:k_part_expand:1" "c2:k_seg_write:1" \
  "c2b:k_gemm_tc:1" "c4:k_dt_bin:1" "c4:k_dt_tile:1" "c4:k_direct_count:1" "c5:k_part_scatter:1" "c5:k_col_stats:1"
python scripts/ncu_summary.py "round 2 dominant kernels (B200, ncu --set full, calibration injected)" gpurun_out/${TAG}_ncu.txt gpurun_out/prof_*.ncu-rep
timeout -s KILL 1800 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; tail -3 gpurun_out/${TAG}_pytest_gpu.log
TCUDB_FUZZ_SEEDS=300 timeout -s KILL 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -k fuzz > gpurun_out/${TAG}_fuzz300.log 2>&1; tail -2 gpurun_out/${TAG}_fuzz300.log
( unset TCUDB_CALIBRATION_VALUES; timeout -s KILL 900 python scripts/selector_sweep.py 4096 16 > gpurun_out/${TAG}_selector_sweep.jsonl 2>/dev/null; \
  timeout -s KILL 900 python scripts/selector_sweep.py 8192 32 >> gpurun_out/${TAG}_selector_sweep.jsonl 2>/dev/null )
python - <<'PY'
import json, os
rows=[json.loads(l) for l in open('gpurun_out/'+os.environ['TAG']+'_selector_sweep.jsonl') if l.startswith('{')]
bad=[r for r in rows if r['selector']!=r['faster'] and r['selector']!='reduce']
print(len(rows), 'points,', len(bad), 'mis-chosen, worst regret', max([r['regret'] for r in rows] or [0]))
PY
unset TCUDB_CALIBRATION_VALUES
bash scripts/gpu_sanitize.sh
