#!/bin/bash
python __graft_entry__.py > /dev/null 2>&1 || exit 1
for c in $@; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv \
      python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
done
