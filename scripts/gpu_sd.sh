#!/bin/bash
# sampled group dictionaries on c5: sample size (2^17 / 2^18 values) x merge blocks (16 / 32)
set -u
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for cfg in "18 16" "17 16" "18 32" "17 32" "16 16"; do
  set -- $cfg
  TCUDB_DICT_SAMPLE_LOG2=$1 TCUDB_SD_BLOCKS=$2 timeout -s KILL 300 python bench.py --config c5 --also "" --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/sd_b.json 2>gpurun_out/sd_b.err
  python -c "import json; d=json.load(open('gpurun_out/sd_b.json')); print('log2=$1 blocks=$2', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()})" || tail -3 gpurun_out/sd_b.err
done
