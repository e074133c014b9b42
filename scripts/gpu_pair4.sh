#!/bin/bash
# fp4 CTA-pair GEMM: parity subset, then c2 bench with the pair kernel vs the 1-CTA kernel
set -u
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -s KILL 300 python -m pytest tests -m gpu -q -x -k "fp4 or e2m1 or c2 or smoke" > gpurun_out/p4_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/p4_pytest.log
for v in 1 0 1 0; do
  TCUDB_GEMM_PAIR4=$v timeout -s KILL 300 python bench.py --config c2 --also "" --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/p4_b_$v.json 2>gpurun_out/p4_b_$v.err
  python -c "import json; d=json.load(open('gpurun_out/p4_b_$v.json')); print('pair=$v', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, round(d['roofline']['achieved'],1), round(d['roofline']['frac'],3))" || tail -5 gpurun_out/p4_b_$v.err
done
