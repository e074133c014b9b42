#!/bin/bash
# the P = 8 key-partitioned intermittent: the collective shim tests repeated (diffs in gpurun_out/collective_diff.jsonl)
set -u
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for i in 1 2 3 4 5 6; do
  TCUDB_DEBUG_BOUNDS=1 timeout -s KILL 600 python -m pytest tests/test_collective_shim.py -m gpu -q -s > gpurun_out/coll_$i.log 2>&1; echo "run $i rc=$?"; tail -1 gpurun_out/coll_$i.log; grep -c "bounds differ" gpurun_out/coll_$i.log
done
