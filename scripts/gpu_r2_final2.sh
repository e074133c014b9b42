#!/bin/bash
# final round-2 evidence: default bench (all configs), launch lists (calibration injected),
# full GPU tests, 300-seed fuzz sweep, selector sweep; every step under a hard-kill timeout
set -u
mkdir -p gpurun_out
TAG=${TAG:-r02g}
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
( time timeout -s KILL 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err ) 2> gpurun_out/${TAG}_bench.time
tail -3 gpurun_out/${TAG}_bench.time
python - <<PY
import json
d=json.load(open('gpurun_out/${TAG}_bench.json'))
print('c2', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['query_roofline']['frac'], d['clocks'], d['e2e']['ms_per_step'])
for c,r in d['configs'].items():
    print(c, round(r['ms_per_step'],3), r['config']['path'], round(r['roofline']['frac'],3), r['query_roofline']['frac'])
PY
export TCUDB_CALIBRATION_VALUES=$(python -c "
import json; c=json.load(open('gpurun_out/${TAG}_bench.json'))['selector_calibration']
print(','.join(repr(c[k]) for k in ('R_i8','R_bf16','R_fp4','BW','R_sp','T_sp0','T_d0')))")
for c in c1 c2 c3 c4 c5 c2b; do
  timeout -s KILL 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/${TAG}_launches_$c.csv \
      python bench.py --config $c --also "" --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
done
unset TCUDB_CALIBRATION_VALUES
timeout -s KILL 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest_gpu.log
TCUDB_FUZZ_SEEDS=300 timeout -s KILL 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -k fuzz > gpurun_out/${TAG}_fuzz300.log 2>&1; echo "fuzz rc=$?"; tail -2 gpurun_out/${TAG}_fuzz300.log
( timeout -s KILL 900 python scripts/selector_sweep.py 4096 16 > gpurun_out/${TAG}_selector_sweep.jsonl 2>/dev/null; \
  timeout -s KILL 900 python scripts/selector_sweep.py 8192 32 >> gpurun_out/${TAG}_selector_sweep.jsonl 2>/dev/null )
python - <<PY
import json
rows=[json.loads(l) for l in open('gpurun_out/${TAG}_selector_sweep.jsonl') if l.startswith('{')]
bad=[r for r in rows if r['selector']!=r['faster'] and r['selector']!='reduce']
print(len(rows), 'points,', len(bad), 'mis-chosen, worst regret', max([r['regret'] for r in rows] or [0]))
PY
