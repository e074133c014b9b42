#!/bin/bash
# final-state ncu --set full captures of each config's dominant kernel (calibration of a normal run injected)
set -u
mkdir -p gpurun_out
rm -f gpurun_out/prof_*.ncu-rep
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -s KILL 300 python bench.py --config c2 --also "" --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pf_c2.json 2>/dev/null
export TCUDB_CALIBRATION_VALUES=$(python -c "
import json; c=json.load(open('gpurun_out/pf_c2.json'))['selector_calibration']
print(','.join(repr(c[k]) for k in ('R_i8','R_bf16','R_fp4','BW','R_sp','T_sp0','T_d0')))")
bash scripts/gpu_prof_multi.sh "c2:k_gemm_tc2:1" "c2:k_seg_write:1" "c4:k_gemm_tc:1" "c3:k_spa_fused:1" "c5:k_part_expand:1"
python scripts/ncu_summary.py "final round-2 state: dominant kernels (B200, ncu --set full, calibration injected)" gpurun_out/r02l_ncu.txt gpurun_out/prof_*.ncu-rep
