#!/bin/bash
# per-kernel launch lists (time + DRAM bytes) for the given configs, calibration constants injected
set -u
mkdir -p gpurun_out
TAG=${TAG:-r02b}
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
export TCUDB_CALIBRATION_VALUES=${TCUDB_CALIBRATION_VALUES:-1.896e15,1.19e15,3.85e15,5.58e12,3.69e10,3.6e-4}
for c in "$@"; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file gpurun_out/${TAG}_launches_$c.csv python bench.py --config $c --also "" --steps 1 --warmup 1 \
     --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
  echo "== $c"; python scripts/launch_table.py gpurun_out/${TAG}_launches_$c.csv 30
done
