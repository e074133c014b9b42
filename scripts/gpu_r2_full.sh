#!/bin/bash
# build, full GPU test suite (hard-killed on a hang), default bench
set -u
mkdir -p gpurun_out
TAG=${TAG:-full}
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -s KILL 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/${TAG}_pytest_gpu.log
if [ "${BENCH:-1}" = 1 ]; then
( time timeout -s KILL 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err ) 2> gpurun_out/${TAG}_bench.time
tail -3 gpurun_out/${TAG}_bench.err
python - <<PY
import json
d=json.load(open('gpurun_out/${TAG}_bench.json'))
print('c2', round(d['ms_per_step'],3), d['roofline']['frac'], d['query_roofline']['frac'], d['clocks'], round(d['e2e']['ms_per_step'],2))
for c,r in d.get('configs',{}).items():
    print(c, round(r['ms_per_step'],3), r['config'].get('path'), round(r['roofline']['frac'],3), r['query_roofline']['frac'], {k: round(v,3) for k,v in r.get('stage_ms',{}).items()})
PY
fi
