#!/bin/bash
# partition scatter geometry sweep on c5: tuples per thread x CTAs per SM (TCUDB_NVCC_EXTRA knobs)
set -u
mkdir -p gpurun_out
for d in "" "-DTCUDB_PART_PER=4 -DTCUDB_PART_MINB=3" "-DTCUDB_PART_PER=4 -DTCUDB_PART_MINB=4" "-DTCUDB_PART_PER=8 -DTCUDB_PART_MINB=2"; do
  TCUDB_NVCC_EXTRA="$d" python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
  timeout -s KILL 300 python bench.py --config c5 --also "" --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pg.json 2>gpurun_out/pg.err
  python -c "import json; d=json.load(open('gpurun_out/pg.json')); print('[$d]', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})" || tail -5 gpurun_out/pg.err
done
