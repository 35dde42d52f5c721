#!/bin/bash
# Round-2 evidence run on one B200 (gpurun): GPU tests, smoke, bench lines for every config,
# the reference arm, the config-3 launch list. Outputs under gpurun_out/r02/ (copied to
# profiles/ by hand).
set -u
mkdir -p gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02/gpu.txt
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout -s KILL 1200 python -m pytest tests -m gpu -q --tb=short -rf --timeout 180 > gpurun_out/r02/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02/tests.log
  python __graft_entry__.py --smoke > gpurun_out/r02/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02/smoke.log
fi
for c in ${CONFIGS:-c3 c2 c1 c4 c5}; do
  python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/r02/bench_$c.json 2> gpurun_out/r02/bench_$c.err
  echo "$c rc=$?"; cut -c1-400 gpurun_out/r02/bench_$c.json
done
if [ "${SKIP_REF:-0}" != "1" ]; then
  python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02/bench_ref_c3.json 2> gpurun_out/r02/bench_ref_c3.err
  echo "ref rc=$?"
fi
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 40 --csv \
    --log-file gpurun_out/r02/launches_c3.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/r02/ncu_launch.log 2>&1
echo "ncu rc=$?"
