#!/bin/bash
# round-2 (late) captures: the CTA-pair e2m1 GEMM on c2 and the c5 encode kernels, plus the c2 launch list
set -u
mkdir -p gpurun_out
rm -f gpurun_out/prof_*.ncu-rep
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout -s KILL 300 python bench.py --config c2 --also "" --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pe_c2.json 2>/dev/null
export TCUDB_CALIBRATION_VALUES=$(python -c "
import json; c=json.load(open('gpurun_out/pe_c2.json'))['selector_calibration']
print(','.join(repr(c[k]) for k in ('R_i8','R_bf16','R_fp4','BW','R_sp','T_sp0','T_d0')))")
timeout -s KILL 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r02e_launches_c2.csv \
    python bench.py --config c2 --also "" --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
bash scripts/gpu_prof_multi.sh "c2:k_gemm_tc2:1" "c5:k_small_distinct:1" "c5:k_group_codes_smem:1" "c5:k_part_scatter:1" "c5:k_col_stats:1" "c5:k_part_hist_all:1"
python scripts/ncu_summary.py "round 2 late: CTA-pair e2m1 GEMM (c2), c5 encode kernels (B200, ncu --set full)" gpurun_out/r02e_ncu.txt gpurun_out/prof_*.ncu-rep
for r in gpurun_out/prof_c5_*.ncu-rep; do ncu -i $r --page source --csv > ${r%.ncu-rep}_src.csv 2>/dev/null; done
