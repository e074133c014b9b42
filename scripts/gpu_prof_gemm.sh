#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 1 -c 1 \
   -o gpurun_out/prof_gemm2_c2 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
TCUDB_GEMM_1CTA=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 | cut -c1-900
