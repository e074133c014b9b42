set -u
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
python -c "
from paper_2112_07552_b200 import Engine
e=Engine(0); print(e.calibration)"
timeout -s KILL 900 python scripts/selector_sweep.py 4096 16 > gpurun_out/sel2.jsonl 2>/dev/null
timeout -s KILL 900 python scripts/selector_sweep.py 8192 32 >> gpurun_out/sel2.jsonl 2>/dev/null
python - <<'PY'
import json
rows=[json.loads(l) for l in open('gpurun_out/sel2.jsonl') if l.startswith('{')]
bad=[r for r in rows if r['selector']!=r['faster'] and r['selector']!='reduce']
print(len(rows), 'points,', len(bad), 'mis-chosen, worst regret', max([r['regret'] for r in rows] or [0]))
for r in bad: print(r['G'], r['K'], r['agg'], r['selector'], r['faster'], round(r['ms_dense'],3), round(r['ms_sparse'],3), round(r['regret'],2))
PY
timeout -s KILL 600 python -m pytest tests -m gpu -q -x -k "calibration or configs_small or selector" 2>&1 | tail -2
for c in c1 c2 c3; do timeout -s KILL 300 python bench.py --config $c --also "" --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],3), d['config'].get('path'))"; done
