#!/bin/bash
# side-stream bucket fill on the sparse path: parity subset, c3 with and without the side stream
set -u
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -k "sparse or c3 or c5 or configs or no_stats or random_tiny or triangle or chain or f2" > gpurun_out/bk_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/bk_pytest.log
for v in 0 1 0 1; do
  TCUDB_NO_SIDE_STREAM=$v timeout -s KILL 300 python bench.py --config c3 --also "" --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bk_b.json 2>gpurun_out/bk_b.err
  python -c "import json; d=json.load(open('gpurun_out/bk_b.json')); print('c3 no_side=$v', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})" || tail -5 gpurun_out/bk_b.err
done
