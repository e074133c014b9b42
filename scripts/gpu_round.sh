#!/bin/bash
# GPU call: build, tests, bench (c2 + optional others), optional ncu.
#   $1: "ncu" (launch list + full GEMM capture) | "launches" (launch list) | "" ; $2: extra configs
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 2>&1 | tail -40 > gpurun_out/t_all.log
tail -5 gpurun_out/t_all.log
for c in c2 $2; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "== $c"; tail -c 2500 gpurun_out/bench_$c.json; tail -3 gpurun_out/bench_$c.err
done
if [ "$1" == "ncu" ] || [ "$1" == "launches" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
      python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
fi
if [ "$1" == "ncu" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 1 -c 1 \
      -o gpurun_out/prof_gemm_c2 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1
  tail -3 gpurun_out/ncu_full.log
fi
