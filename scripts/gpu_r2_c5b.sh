#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "hash or c5 or configs_small" > gpurun_out/pytest_c5b.log 2>&1; tail -3 gpurun_out/pytest_c5b.log
for m in 0 1; do
  TCUDB_HASHPART_HISTSCAN=$m timeout 600 python bench.py --config c5 --also "" --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_c5_$m.json 2>gpurun_out/b_c5_$m.err
  python -c "import json; d=json.load(open('gpurun_out/b_c5_$m.json')); print('c5 histscan=$m', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})" || tail -3 gpurun_out/b_c5_$m.err
done
TCUDB_CALIBRATE=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5b.csv python bench.py --config c5 --also "" --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/launches_c5b.csv 14
