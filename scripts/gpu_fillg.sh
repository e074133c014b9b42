#!/bin/bash
# g column in its own vectorised pass: parity subset, c2 / c4 / c5 with and without
set -u
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -k "c2 or c4 or c5 or configs or no_stats or random_tiny or fused or block or hash_part or int64 or f2" > gpurun_out/fg_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/fg_pytest.log
for c in c2 c4 c5; do for v in 0 1 0 1; do
  TCUDB_NO_FILL_G=$v timeout -s KILL 300 python bench.py --config $c --also "" --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/fg_b.json 2>gpurun_out/fg_b.err
  python -c "import json; d=json.load(open('gpurun_out/fg_b.json')); print('$c no_fill_g=$v', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})" || tail -5 gpurun_out/fg_b.err
done; done
