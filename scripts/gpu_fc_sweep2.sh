#!/bin/bash
# f1 fused compaction: compaction warps x raster band height on c2 (query ms), vs separate
set -u
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout -s KILL 300 python bench.py --config c2 --also "" --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/fc_sep.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/fc_sep.json')); print('separate', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})"
for W in 4 8 12; do
  TCUDB_NVCC_EXTRA="-DTCUDB_CMP_WARPS=$W" python -c "from paper_2112_07552_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  for G in 2 4 8 16; do
    TCUDB_FUSED_COMPACT=1 TCUDB_GEMM_GROUP_M=$G timeout -s KILL 300 python bench.py --config c2 --also "" --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/fc_${W}_$G.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/fc_${W}_$G.json')); print('W=$W G=$G', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, d['config'].get('fused_compact'))" 2>/dev/null || echo "W=$W G=$G failed"
  done
done
TCUDB_FUSED_COMPACT=1 timeout -s KILL 300 python -m pytest tests -m gpu -q -x -k "fused_compaction" 2>&1 | tail -2
