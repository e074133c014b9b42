#!/bin/bash
# GPU call: build, tests, bench, ncu launch list + full capture of the GEMM (c2).
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 2>&1 | tail -40 > gpurun_out/t_all.log
tail -5 gpurun_out/t_all.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
tail -c 3000 gpurun_out/bench_c2.json; tail -5 gpurun_out/bench_c2.err
if [ "$1" == "ncu" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
      python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 1 -c 1 \
      -o gpurun_out/prof_gemm_c2 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1
  tail -3 gpurun_out/ncu_full.log
fi
