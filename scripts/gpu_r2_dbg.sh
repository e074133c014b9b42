#!/bin/bash
set -u
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "fused_direct" > gpurun_out/dbg_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/dbg_pytest.log
TCUDB_LAZY_CODES=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests -m gpu -q -x -k "fused_direct and signed_split" > gpurun_out/dbg_san.log 2>&1; echo "san rc=$?"; grep -v '^=========     ' gpurun_out/dbg_san.log | head -40
export TCUDB_CALIBRATION_VALUES=1.896e15,1.19e15,3.85e15,5.58e12,3.69e10,3.6e-4
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file gpurun_out/dbg_launches_c4.csv python bench.py --config c4 --also "" --steps 1 --warmup 0 \
     --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/dbg_launches_c4.csv 20
