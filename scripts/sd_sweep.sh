python __graft_entry__.py > gpurun_out/build.log 2>&1
export TCUDB_CALIBRATION_VALUES=1.896e15,1.19e15,3.85e15,5.58e12,3.69e10,3.6e-4
for nb in 2 4 8 16; do for li in 0 1; do
TCUDB_SD_LIST=$li TCUDB_SD_BLOCKS=$nb timeout -s KILL 200 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_small_distinct|k_sd_merge" \
     --log-file gpurun_out/sd_$nb_$li.csv python bench.py --config c5 --also "" --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
echo "nb=$nb list=$li"; python scripts/launch_table.py gpurun_out/sd_$nb_$li.csv 3
done; done
