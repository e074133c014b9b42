#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2f.log 2>&1; tail -12 gpurun_out/pytest_gpu_r2f.log
for c in c2 c2b c4s c5 c3; do
  timeout 600 python bench.py --config $c --also "" --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
  python -c "import json; d=json.load(open('gpurun_out/b_$c.json')); print('$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, d['config']['path'], d['roofline']['frac'])" || tail -3 gpurun_out/b_$c.err
done
