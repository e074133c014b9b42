#!/bin/bash
# round 2 first call: build, accumulation-precision probe, GPU tests at the round-1 state
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python scripts/precision_probe.py gpurun_out/precision_probe.json > gpurun_out/precision_probe.log 2>&1
tail -20 gpurun_out/precision_probe.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r2a.log 2>&1
tail -5 gpurun_out/pytest_gpu_r2a.log
