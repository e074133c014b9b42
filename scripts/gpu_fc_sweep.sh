#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests -m gpu -q -x --timeout 90 -k "fused_compaction" 2>&1 | tail -2
run() {
  timeout 300 env "$@" python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/sw.json 2> gpurun_out/sw.err
  python -c "
import json; d=json.load(open('gpurun_out/sw.json')); print('$*', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items() if v > 0})"
}
run TCUDB_NO_FUSED_COMPACT=1
run TCUDB_NO_FUSED_COMPACT=0
for g in 2 8; do run TCUDB_GEMM_GROUP_M=$g; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -c 1 -o gpurun_out/prof_c2_fused -f \
   env TCUDB_GEMM_GROUP_M=2 python bench.py --config c2 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_fused.log 2>&1
tail -1 gpurun_out/ncu_fused.log
