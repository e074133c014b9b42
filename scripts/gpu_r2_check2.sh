#!/bin/bash
# c5 timing with the cheaper statistics pass, 300-seed fuzz at the current state
set -u
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for c in c5 c2; do timeout -s KILL 300 python bench.py --config $c --also "" --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})"; done
export TCUDB_CALIBRATION_VALUES=1.896e15,1.19e15,3.85e15,5.58e12,3.69e10,3.6e-4
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file gpurun_out/k2_launches_c5.csv python bench.py --config c5 --also "" --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/k2_launches_c5.csv 8
unset TCUDB_CALIBRATION_VALUES
TCUDB_FUZZ_SEEDS=300 timeout -s KILL 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -k fuzz > gpurun_out/r02_fuzz300_final.log 2>&1; tail -2 gpurun_out/r02_fuzz300_final.log
