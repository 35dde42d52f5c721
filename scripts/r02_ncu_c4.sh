#!/bin/bash
# Round-2 ncu evidence for config 4's recurrence (fused gate-cluster k_lstm_seq) at T = 8.
set -u
mkdir -p gpurun_out/r02

T=8 python scripts/c4_probe.py > gpurun_out/r02/plain_c4.log 2>&1 || { cat gpurun_out/r02/plain_c4.log; exit 1; }
cat gpurun_out/r02/plain_c4.log
T=8 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02/launches_c4_T8.csv python scripts/c4_probe.py > gpurun_out/r02/ncu_launch_c4.log 2>&1
echo "launch list rc=$?"
T=8 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lstm_seq -s 2 -c 1 \
    -o gpurun_out/r02/prof_lstm_seq -f python scripts/c4_probe.py > gpurun_out/r02/ncu_full_c4.log 2>&1
echo "ncu full rc=$?"
ncu -i gpurun_out/r02/prof_lstm_seq.ncu-rep --page details > gpurun_out/r02/lstm_seq_c4_ncu_details.txt 2>&1
