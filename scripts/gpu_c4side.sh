#!/bin/bash
# c4 fused fills on two streams: parity subset, c4 / c4s with and without the side stream
set -u
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -k "fused_direct or c4 or float or configs_small or no_stats" > gpurun_out/c4s_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/c4s_pytest.log
for c in c4 c4s; do for v in 0 1 0 1; do
  TCUDB_NO_SIDE_STREAM=$v timeout -s KILL 300 python bench.py --config $c --also "" --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/c4s_b.json 2>gpurun_out/c4s_b.err
  python -c "import json; d=json.load(open('gpurun_out/c4s_b.json')); print('$c no_side=$v', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})" || tail -3 gpurun_out/c4s_b.err
done; done
