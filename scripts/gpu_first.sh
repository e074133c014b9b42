#!/bin/bash
# first GPU call: build, GEMM unit tests under a hard timeout, then the rest.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 180 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm" --timeout 60 2>&1 | tail -30 | tee gpurun_out/t_gemm.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -20 | tee gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -x 2>&1 | tail -40 | tee gpurun_out/t_all.log
