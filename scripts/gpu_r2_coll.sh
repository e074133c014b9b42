#!/bin/bash
# round 2: collective path at P=2/4/8 (in-process communicator), GPU suite, default bench
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_collective_shim.py -x -q > gpurun_out/pytest_shim.log 2>&1
tail -25 gpurun_out/pytest_shim.log
timeout 1800 python -m pytest tests -m gpu -q --deselect tests/test_collective_shim.py > gpurun_out/pytest_gpu_r2c.log 2>&1
tail -8 gpurun_out/pytest_gpu_r2c.log
( time timeout 900 python bench.py > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.err ) 2> gpurun_out/bench_r2c.time
cat gpurun_out/bench_r2c.time; tail -3 gpurun_out/bench_r2c.err
