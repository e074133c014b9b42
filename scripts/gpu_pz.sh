#!/bin/bash
# pre-zeroed e2m1 operands + side-stream fills: parity subset, c2 / c2b / c1 bench with and without
set -u
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -k "fp4 or e2m1 or c2 or configs_small or no_stats or random_tiny or fused or block or count" > gpurun_out/pz_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pz_pytest.log
for c in c2 c2b c1; do for v in 0 1 0 1; do
  TCUDB_NO_PREZERO=$v timeout -s KILL 300 python bench.py --config $c --also "" --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pz_b.json 2>gpurun_out/pz_b.err
  python -c "import json; d=json.load(open('gpurun_out/pz_b.json')); print('$c no_prezero=$v', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})" || tail -5 gpurun_out/pz_b.err
done; done
