#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 200 python -m pytest tests/test_gpu_parity.py -x -q -k "fp4" --timeout 60 2>&1 | tail -25
