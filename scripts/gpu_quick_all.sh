#!/bin/bash
# build, a GPU test subset (-k expr in $1, "" = all), then bench of each config in $2..
set -u
mkdir -p gpurun_out
TAG=${TAG:-q}
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
if [ "$1" = "ALL" ]; then
  timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
elif [ -n "$1" ]; then
  timeout -s KILL 900 python -m pytest tests -m gpu -q -x -k "$1" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
fi
shift
for c in "$@"; do
  timeout -s KILL 600 python bench.py --config $c --also "" --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${TAG}_b_$c.json 2>gpurun_out/${TAG}_b_$c.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_b_$c.json')); print('$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, d['config'].get('path'), round(d['roofline']['frac'],3))" || tail -5 gpurun_out/${TAG}_b_$c.err
done
