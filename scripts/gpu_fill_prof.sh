#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
TCUDB_FILL_PASSES=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fill_bf16_rows -c 1 -o gpurun_out/prof_c4_fill_rows -f \
  python bench.py --config c4 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
TCUDB_FILL_PASSES=3 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/c4_rows_launches.csv python bench.py --config c4 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
true
