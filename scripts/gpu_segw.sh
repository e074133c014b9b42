#!/bin/bash
# ordered compaction with an affine h dictionary: segments per warp iteration (TCUDB_SEGW_P)
set -u
mkdir -p gpurun_out
for P in 2 3 4; do
  TCUDB_NVCC_EXTRA="-DTCUDB_SEGW_P=$P" python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
  if [ $P = 2 ]; then timeout -s KILL 600 python -m pytest tests -m gpu -q -x -k "c2 or c4 or configs_small or fused or random_tiny" > gpurun_out/sw_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/sw_pytest.log; fi
  for c in c2 c4; do
    timeout -s KILL 300 python bench.py --config $c --also "" --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/sw_b.json 2>gpurun_out/sw_b.err
    python -c "import json; d=json.load(open('gpurun_out/sw_b.json')); print('P=$P $c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})" || tail -5 gpurun_out/sw_b.err
  done
done
