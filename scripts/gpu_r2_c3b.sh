#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "sparse_spa or configs_full or fuzz or c3" > gpurun_out/pytest_c3b.log 2>&1; tail -3 gpurun_out/pytest_c3b.log
timeout 600 python bench.py --config c3 --also "" --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_c3.json 2>gpurun_out/b_c3.err
python -c "import json; d=json.load(open('gpurun_out/b_c3.json')); print('c3', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, d['roofline']['frac'], d['roofline']['avg_launch_ms'])"
TCUDB_CALIBRATE=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3b.csv python bench.py --config c3 --also "" --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/launches_c3b.csv 20
