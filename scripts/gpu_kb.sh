#!/bin/bash
python __graft_entry__.py > /dev/null 2>&1 || exit 1
TCUDB_GEMM_KB=64 timeout 200 python -m pytest tests/test_gpu_parity.py -x -q -k "gemm or fp4 or c4" --timeout 60 2>&1 | tail -2
for kb in 128 64; do
  TCUDB_GEMM_KB=$kb timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kb=$kb c2', round(d['ms_per_step'],3), round(d['stage_ms']['ms_gemm'],3), round(d['roofline']['achieved']))"
  TCUDB_NO_FP4=1 TCUDB_GEMM_KB=$kb timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kb=$kb c2 i8', round(d['ms_per_step'],3), round(d['stage_ms']['ms_gemm'],3), round(d['roofline']['achieved']))"
  TCUDB_GEMM_KB=$kb timeout 300 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kb=$kb c4', round(d['ms_per_step'],3), round(d['stage_ms']['ms_gemm'],3), round(d['roofline']['achieved']))"
done
