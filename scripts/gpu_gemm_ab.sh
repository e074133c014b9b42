#!/bin/bash
# GEMM A/B: pair kernel vs 1-CTA kernel on c2 (bench stage times)
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k gemm --timeout 60 2>&1 | tail -3
for v in 0 1; do
  TCUDB_GEMM_PAIR=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab_$v.json
  python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print('pair=$v', d['ms_per_step'], d['stage_ms'], d['roofline']['achieved'])"
done
