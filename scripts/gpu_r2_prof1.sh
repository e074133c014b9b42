#!/bin/bash
# ncu --set full of selected kernels: "config:regex:count" triples, summary to gpurun_out/${TAG}_ncu.txt
set -u
TAG=${TAG:-p}
export TCUDB_CALIBRATION_VALUES=${TCUDB_CALIBRATION_VALUES:-1.896e15,1.19e15,3.85e15,5.58e12,3.69e10,3.6e-4}
rm -f gpurun_out/prof_*.ncu-rep
bash scripts/gpu_prof_multi.sh "$@"
python scripts/ncu_summary.py "$TAG" gpurun_out/${TAG}_ncu.txt gpurun_out/prof_*.ncu-rep
cat gpurun_out/${TAG}_ncu.txt
