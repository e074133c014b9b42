#!/bin/bash
# c3 iteration: sparse GPU tests, c3 bench x2, launch list
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
[ "$1" = "test" ] && timeout 900 python -m pytest tests -m gpu -x -q -k "spa or sparse or fuzz or config or tri or chain" 2>&1 | tail -3
for i in 1 2; do
  timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); print('c3', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, round(d['roofline']['avg_launch_ms'],3))"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/c3_try_launches.csv python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
[ -n "$2" ] && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$2" -c 1 -o gpurun_out/prof_c3_try -f \
  python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
true
