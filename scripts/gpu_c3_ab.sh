#!/bin/bash
# c3 A/B of an env switch: $1 = VAR=value for the B arm
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "spa or sparse or fuzz or config or tri or chain" 2>&1 | tail -2
for E in X=0 $1 X=0 $1; do
  env $E timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); print('$E', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, round(d['roofline']['avg_launch_ms'],3))"
done
