#!/bin/bash
# build, GPU tests (optionally filtered by $1), then benches of the configs in $2
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
if [ -n "$1" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x --timeout 400 -k "$1" 2>&1 | tail -30 > gpurun_out/t_quick.log
  tail -8 gpurun_out/t_quick.log
fi
for c in $2; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python - <<PY
import json
d = json.load(open("gpurun_out/bench_$c.json"))
print("$c", round(d["ms_per_step"], 3), {k: round(v, 3) for k, v in d["stage_ms"].items()}, d["config"].get("path"), d["dtype"])
PY
  tail -2 gpurun_out/bench_$c.err
done
