#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "sparse_spa or configs_full or c3 or triangles" > gpurun_out/pytest_c3.log 2>&1; tail -3 gpurun_out/pytest_c3.log
for h in 0 1; do
  TCUDB_SPA_NO_HUB=$h timeout 600 python bench.py --config c3 --also "" --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_c3_$h.json 2>gpurun_out/b_c3_$h.err
  python -c "import json; d=json.load(open('gpurun_out/b_c3_$h.json')); print('c3 nohub=$h', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, d['roofline']['spa_mode'], d['roofline']['frac'])" || tail -3 gpurun_out/b_c3_$h.err
done
TCUDB_CALIBRATE=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --also "" --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/launches_c3.csv 14
bash scripts/gpu_prof_multi.sh "c3:k_spa_fused:1"
ncu -i gpurun_out/prof_c3_k_spa_fused.ncu-rep --page source --csv --print-source sass > gpurun_out/c3_spa_source.csv 2>/dev/null; ls -la gpurun_out/c3_spa_source.csv
