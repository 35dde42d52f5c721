#!/bin/bash
# Round-2 ncu evidence on one B200 (after the plain command has exited 0):
#   1. --set full capture of one steady launch of the row-tile kernel (config 3) -> .ncu-rep + details
#   2. steady-state DRAM traffic range of the row-tile kernel (12 launches, no cache flush)
#   3. per-GPU shard sweep of config 3 (bench --shard-of N, both row kernels)
set -u
mkdir -p gpurun_out/r02
python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02/plain_c3.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_tc_rows_reuse -s 14 -c 1 \
    -o gpurun_out/r02/prof_rows_c3 -f python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/r02/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i gpurun_out/r02/prof_rows_c3.ncu-rep --page details > gpurun_out/r02/rows_c3_ncu_details.txt 2>&1
ncu --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    -k regex:k_tc_rows_reuse -s 12 -c 12 --csv --log-file gpurun_out/r02/traffic_c3_rows.csv \
    python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02/ncu_traffic.log 2>&1
echo "ncu traffic rc=$?"
bash scripts/ab_shard.sh > gpurun_out/r02/shard_sweep.txt 2>&1; cat gpurun_out/r02/shard_sweep.txt
