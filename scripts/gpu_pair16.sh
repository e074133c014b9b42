#!/bin/bash
# CTA-pair kernel for kind::f16 / kind::i8 (TCUDB_GEMM_PAIR=1) vs the 1-CTA kernel on c4 / c4s
set -u
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
TCUDB_GEMM_PAIR=1 timeout -s KILL 600 python -m pytest tests -m gpu -q -x -k "c4 or bf16 or gemm or i8" > gpurun_out/p16_pytest.log 2>&1; echo "pytest(pair) rc=$?"; tail -3 gpurun_out/p16_pytest.log
for c in c4 c4s; do
for v in 1 0 1 0; do
  TCUDB_GEMM_PAIR=$v timeout -s KILL 300 python bench.py --config $c --also "" --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/p16_b_$v.json 2>gpurun_out/p16_b_$v.err
  python -c "import json; d=json.load(open('gpurun_out/p16_b_$v.json')); print('$c pair=$v', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, round(d['roofline']['achieved'],1), round(d['roofline']['frac'],3))" || tail -5 gpurun_out/p16_b_$v.err
done
done
