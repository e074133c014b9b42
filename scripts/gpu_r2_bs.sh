#!/bin/bash
# block-sparse + c5 changes: targeted tests, then the whole GPU suite, benches of c5 / c2b / c2
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_block_sparse.py -q -x > gpurun_out/pytest_bs.log 2>&1; tail -15 gpurun_out/pytest_bs.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2e.log 2>&1; tail -8 gpurun_out/pytest_gpu_r2e.log
for c in c5 c2b c2; do
  timeout 600 python bench.py --config $c --also "" --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
  python -c "import json; d=json.load(open('gpurun_out/b_$c.json')); print('$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, d['config']['path'], d['roofline']['frac'])" || tail -3 gpurun_out/b_$c.err
done
TCUDB_BLOCK_SPARSE=0 timeout 600 python bench.py --config c2b --also "" --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_c2b_off.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/b_c2b_off.json')); print('c2b bs-off', round(d['ms_per_step'],3), d['config']['path'])"
