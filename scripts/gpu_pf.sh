#!/bin/bash
# persistent prefetching partition scatter (COUNT): parity subset, c5 with and without
set -u
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -k "hash_part or c5 or sampled or no_stats or configs_small or collective" > gpurun_out/pf_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pf_pytest.log
for v in 1 0 1 0; do
  TCUDB_PART_PF=$v timeout -s KILL 300 python bench.py --config c5 --also "" --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pf_b.json 2>gpurun_out/pf_b.err
  python -c "import json; d=json.load(open('gpurun_out/pf_b.json')); print('c5 pf=$v', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})" || tail -3 gpurun_out/pf_b.err
done
