#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests -m gpu -q -x --timeout 90 -k "fused_compaction" 2>&1 | tail -25 > gpurun_out/t_fc.log
tail -25 gpurun_out/t_fc.log
if grep -q "passed" gpurun_out/t_fc.log && ! grep -q "failed" gpurun_out/t_fc.log; then
  timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -5
  for c in c2; do
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
    python -c "
import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, d['roofline']['frac'])"
  done
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
      python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
fi
