#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tc|k_seg_write" -s 2 -c 2 \
   -o gpurun_out/prof_c2_v5 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
