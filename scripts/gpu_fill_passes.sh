#!/bin/bash
# c4 fill: binned (default) vs row-range passes (TCUDB_FILL_PASSES)
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
run() { env $1 timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); print('$1', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})"; }
run X=0; run TCUDB_FILL_PASSES=3

TCUDB_FILL_PASSES=${1:-3} timeout 600 python -m pytest tests -m gpu -x -q -k "c4 or float or bf16 or fuzz" 2>&1 | tail -2
