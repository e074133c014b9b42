#!/bin/bash
# last validation + evidence: smoke, full GPU suite, default bench, c2 / c3 launch lists
set -u
mkdir -p gpurun_out
TAG=${TAG:-r02i}
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -s KILL 300 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest_gpu.log
timeout -s KILL 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python - <<PY
import json
d=json.load(open('gpurun_out/${TAG}_bench.json'))
print('c2', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['query_roofline']['frac'], d['clocks'], d['e2e']['ms_per_step'], d['gpu_launches'])
for c,r in d['configs'].items():
    print(c, round(r['ms_per_step'],3), r['config']['path'], round(r['roofline']['frac'],3), r['query_roofline']['frac'])
PY
export TCUDB_CALIBRATION_VALUES=$(python -c "
import json; c=json.load(open('gpurun_out/${TAG}_bench.json'))['selector_calibration']
print(','.join(repr(c[k]) for k in ('R_i8','R_bf16','R_fp4','BW','R_sp','T_sp0','T_d0')))")
for c in c1 c2 c3 c4 c5; do
  timeout -s KILL 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/${TAG}_launches_$c.csv \
      python bench.py --config $c --also "" --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
done
