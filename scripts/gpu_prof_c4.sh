#!/bin/bash
# c4 encode/fill kernels: one full ncu capture each of the named kernels
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
K=${1:-"k_bin_scatter|k_bin_split|k_col_stats"}
C=${2:-3}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 0 -c $C \
   -o gpurun_out/prof_c4_fill -f python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
