#!/bin/bash
set -u
mkdir -p gpurun_out
TAG=${TAG:-c4}
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -s KILL 600 python -m pytest tests -m gpu -q -x -k "fused_direct or c4_full" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
for c in c4 c4s; do
timeout -s KILL 300 python bench.py --config $c --also "" --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${TAG}_b_$c.json 2>gpurun_out/${TAG}_b_$c.err
python -c "import json; d=json.load(open('gpurun_out/${TAG}_b_$c.json')); print('$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, d['query_roofline']['frac'])" || tail -5 gpurun_out/${TAG}_b_$c.err
done
export TCUDB_CALIBRATION_VALUES=1.896e15,1.19e15,3.85e15,5.58e12,3.69e10,3.6e-4
for c in c4 c4s; do
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file gpurun_out/${TAG}_launches_$c.csv python bench.py --config $c --also "" --steps 1 --warmup 0 \
     --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/${TAG}_launches_$c.csv 12
done
