#!/bin/bash
# one full ncu capture of the kernels matching $2 in config $1 (first $3 launches)
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s 0 -c ${3:-1} \
   -o gpurun_out/prof_$1 -f python bench.py --config $1 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_full_$1.log 2>&1
tail -2 gpurun_out/ncu_full_$1.log
