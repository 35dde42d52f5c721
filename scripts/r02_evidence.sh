#!/bin/bash
# Round-2 evidence run on one B200 (gpurun): bench lines for every config, the reference arm,
# the config-3 launch list and clocks. Outputs under gpurun_out/r02/ (copied to profiles/ by hand).
set -u
mkdir -p gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02/gpu.txt
for c in c3 c2 c1 c4 c5; do
  python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/r02/bench_$c.json 2> gpurun_out/r02/bench_$c.err
  echo "$c rc=$?"
done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02/bench_ref_c3.json 2> gpurun_out/r02/bench_ref_c3.err
echo "ref rc=$?"
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 40 --csv \
    --log-file gpurun_out/r02/launches_c3.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/r02/ncu_launch.log 2>&1
echo "ncu rc=$?"
