#!/bin/bash
# full ncu captures of selected kernels: args are "config:regex:count" triples
# (the create-time calibration would otherwise be the first GEMM / sparse launches the regex
#  matches, and its timing under ncu is distorted: pass the constants of a normal run in
#  TCUDB_CALIBRATION_VALUES, else the compiled defaults are used)
mkdir -p gpurun_out
if [ -z "$TCUDB_CALIBRATION_VALUES" ]; then export TCUDB_CALIBRATE=0; fi
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for spec in "$@"; do
  IFS=: read c re n <<< "$spec"
  tag=$(echo "$re" | tr -c 'a-zA-Z0-9_\n' '_')
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"$re" -c ${n:-1} \
     -o gpurun_out/prof_${c}_${tag} -f python bench.py --config $c --also "" --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 \
     > gpurun_out/ncu_${c}_${tag}.log 2>&1
  tail -2 gpurun_out/ncu_${c}_${tag}.log
done
