#!/bin/bash
# re-entry check: build, default bench (all configs), full GPU test suite
set -u
mkdir -p gpurun_out
TAG=${TAG:-re}
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -s KILL 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python - <<PY
import json
d=json.load(open('gpurun_out/${TAG}_bench.json'))
print('c2', round(d['ms_per_step'],3), d['roofline']['frac'], d['query_roofline']['frac'], d['clocks'])
for c,r in d['configs'].items():
    print(c, round(r['ms_per_step'],3), r['config']['path'], round(r['roofline']['frac'],3), r['query_roofline']['frac'])
PY
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest_gpu.log
