#!/bin/bash
python __graft_entry__.py > /dev/null 2>&1 || exit 1
timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm" --timeout 60 2>&1 | tail -2
for gm in 0 8 16 40 80; do
  for cfg in c2; do
    TCUDB_GEMM_GROUP_M=$gm timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gm=$gm $cfg', round(d['ms_per_step'],3), round(d['stage_ms']['ms_gemm'],3), round(d['roofline']['achieved']))"
    TCUDB_NO_FP4=1 TCUDB_GEMM_GROUP_M=$gm timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gm=$gm $cfg i8', round(d['ms_per_step'],3), round(d['stage_ms']['ms_gemm'],3), round(d['roofline']['achieved']))"
  done
done
