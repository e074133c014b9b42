#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_block_sparse.py tests/test_collective_shim.py -q -x -k "block or key_part" > gpurun_out/pytest_bs2.log 2>&1; tail -15 gpurun_out/pytest_bs2.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "configs or fuzz or fp4 or c4" > gpurun_out/pytest_sub.log 2>&1; tail -3 gpurun_out/pytest_sub.log
for c in c2 c2b; do
 for bs in auto 0; do
  if [ $bs = auto ]; then unset TCUDB_BLOCK_SPARSE; else export TCUDB_BLOCK_SPARSE=0; fi
  timeout 600 python bench.py --config $c --also "" --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
  python -c "import json; d=json.load(open('gpurun_out/b_$c.json')); print('$c bs=$bs', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, d['config']['path'], d['roofline']['frac'])" || tail -3 gpurun_out/b_$c.err
 done
done
unset TCUDB_BLOCK_SPARSE
TCUDB_CALIBRATE=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2b.csv python bench.py --config c2b --also "" --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/launches_c2b.csv 14
