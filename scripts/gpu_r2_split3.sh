#!/bin/bash
set -u
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "fuzz" > gpurun_out/s3_fuzz.log 2>&1; echo "fuzz rc=$?"; tail -3 gpurun_out/s3_fuzz.log
timeout -s KILL 300 python scripts/precision_probe.py gpurun_out/r02_precision_probe.json > gpurun_out/s3_probe.log 2>&1; grep split3 gpurun_out/s3_probe.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q > gpurun_out/s3_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s3_pytest_gpu.log
timeout -s KILL 300 python bench.py --config c4s --also "" --steps 5 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/s3_c4s.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/s3_c4s.json')); print('c4s', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})"
