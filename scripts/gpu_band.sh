#!/bin/bash
# banded GEMM ‖ compaction on c2: parity subset, then bench with 0 / 2 / 4 / 8 bands and write-grid caps
set -u
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -s KILL 400 python -m pytest tests -m gpu -q -x -k "fp4 or e2m1 or c2 or smoke or count" > gpurun_out/band_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/band_pytest.log
run() {
  env "$@" timeout -s KILL 300 python bench.py --config c2 --also "" --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/band_b.json 2>gpurun_out/band_b.err
  python -c "import json; d=json.load(open('gpurun_out/band_b.json')); print('$*', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items()}, round(d['roofline']['frac'],3))" || tail -5 gpurun_out/band_b.err
}
run TCUDB_BAND_COMPACT=0
run TCUDB_BAND_COMPACT=4
run TCUDB_BAND_COMPACT=2
run TCUDB_BAND_COMPACT=8
run TCUDB_BAND_COMPACT=4 TCUDB_BAND_GRID=296
run TCUDB_BAND_COMPACT=4 TCUDB_BAND_GRID=74
run TCUDB_BAND_COMPACT=0
run TCUDB_BAND_COMPACT=4
