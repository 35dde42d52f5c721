#!/bin/bash
# Round-2 ncu evidence for config 2 (general path) after the regeneration-overlap change:
# launch list, --set full of the hi|lo GEMM and of k_regen_wt, steady-state DRAM traffic.
set -u
mkdir -p gpurun_out/r02
B="python bench.py --config c2 --steps 6 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/r02/plain_c2.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -s 10 -c 24 --csv \
    --log-file gpurun_out/r02/launches_c2.csv $B > gpurun_out/r02/ncu_launch_c2.log 2>&1; echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_tc_xgemm -s 8 -c 1 \
    -o gpurun_out/r02/prof_xgemm_c2 -f $B > gpurun_out/r02/ncu_full_c2.log 2>&1; echo "ncu full rc=$?"
ncu -i gpurun_out/r02/prof_xgemm_c2.ncu-rep --page details > gpurun_out/r02/xgemm_c2_ncu_details.txt 2>&1
ncu --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    -k regex:k_tc_xgemm -s 8 -c 12 --csv --log-file gpurun_out/r02/traffic_c2_xgemm.csv \
    $B > gpurun_out/r02/ncu_traffic_c2.log 2>&1; echo "ncu traffic rc=$?"
