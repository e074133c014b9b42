#!/bin/bash
# final validation: build, smoke(), full GPU suite, default bench
set -u
mkdir -p gpurun_out
TAG=${TAG:-r02h}
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -s KILL 300 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/${TAG}_smoke.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest_gpu.log
timeout -s KILL 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python - <<PY
import json
d=json.load(open('gpurun_out/${TAG}_bench.json'))
print('c2', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['query_roofline']['frac'], d['clocks'], d['e2e']['ms_per_step'], d['gpu_launches'])
for c,r in d['configs'].items():
    print(c, round(r['ms_per_step'],3), r['config']['path'], round(r['roofline']['frac'],3), r['query_roofline']['frac'])
PY
