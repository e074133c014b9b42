#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 400 python -m pytest tests -m gpu -q -x --timeout 120 -k "hash_partitioned" 2>&1 | tail -25 > gpurun_out/t_hp.log
tail -25 gpurun_out/t_hp.log
if grep -q "passed" gpurun_out/t_hp.log && ! grep -q "failed" gpurun_out/t_hp.log; then
  timeout 300 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_c5.json')); print('c5', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, d['roofline'])"
  tail -3 gpurun_out/bench_c5.err
  bash scripts/gpu_launches.sh c5
  timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -3
fi
