#!/bin/bash
# round-2 re-entry check: build, GPU tests, default bench
set -u
mkdir -p gpurun_out
TAG=${TAG:-r02a}
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${TAG}_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/${TAG}_pytest_gpu.log
( time timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err ) 2> gpurun_out/${TAG}_bench.time
tail -3 gpurun_out/${TAG}_bench.time; tail -3 gpurun_out/${TAG}_bench.err
python - <<PY
import json
d=json.load(open('gpurun_out/${TAG}_bench.json'))
print('c2', round(d['ms_per_step'],3), d['roofline']['frac'], d['query_roofline']['frac'], d['clocks'], d.get('e2e'))
for c,r in d.get('configs',{}).items():
    print(c, round(r['ms_per_step'],3), r['config'].get('path'), round(r['roofline']['frac'],3), r['query_roofline']['frac'])
PY
