#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r2g.log 2>&1; tail -6 gpurun_out/pytest_gpu_r2g.log
for c in c4 c4s c3; do
  timeout 600 python bench.py --config $c --also "" --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err
  python -c "import json; d=json.load(open('gpurun_out/b_$c.json')); print('$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, d['roofline']['frac'])" || tail -3 gpurun_out/b_$c.err
done
bash scripts/gpu_prof_multi.sh "c3:k_spa_fused:1"
ncu -i gpurun_out/prof_c3_k_spa_fused.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/c3_spa_source2.csv 2>gpurun_out/c3_src.err; ls -la gpurun_out/c3_spa_source2.csv; tail -2 gpurun_out/c3_src.err
