#!/bin/bash
# c4 fill modes: parity + bench per mode, launch list of the tiled mode
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fill or c4" > gpurun_out/pytest_c4fill.log 2>&1; tail -3 gpurun_out/pytest_c4fill.log
for m in tiled range binned; do
  TCUDB_FILL_MODE=$m timeout 600 python bench.py --config c4 --also "" --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/c4_$m.json 2>gpurun_out/c4_$m.err
  python -c "import json; d=json.load(open('gpurun_out/c4_$m.json')); print('$m', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4_tiled.csv python bench.py --config c4 --also "" --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/launches_c4_tiled.csv 12
