#!/bin/bash
# GEMM abort on an overflowed optimistic fill + per-plane dense fixed cost: parity subset, selector sweep, c1-c5 bench
set -u
mkdir -p gpurun_out
TAG=${TAG:-r02j}
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x -k "fp4 or u8 or wide or dup or configs or random_tiny or sum or count or fused or block" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${TAG}_pytest.log
( timeout -s KILL 900 python scripts/selector_sweep.py 4096 16 > gpurun_out/${TAG}_selector_sweep.jsonl 2>/dev/null; \
  timeout -s KILL 900 python scripts/selector_sweep.py 8192 32 >> gpurun_out/${TAG}_selector_sweep.jsonl 2>/dev/null )
python - <<PY
import json
rows=[json.loads(l) for l in open('gpurun_out/${TAG}_selector_sweep.jsonl') if l.startswith('{')]
bad=[r for r in rows if r['selector']!=r['faster'] and r['selector']!='reduce']
print(len(rows), 'points,', len(bad), 'mis-chosen, worst regret', max([r['regret'] for r in rows] or [0]))
for r in bad: print('  ', r['G'], r['K'], r['agg'], r['ms_dense'], r['ms_sparse'], r['ms_auto'], r['selector'], r['regret'])
PY
for c in c1 c2 c3 c4 c5; do
  timeout -s KILL 300 python bench.py --config $c --also "" --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${TAG}_b.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_b.json')); print('$c', round(d['ms_per_step'],3), d['config']['path'])"
done
