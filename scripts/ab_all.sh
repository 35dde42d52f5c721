#!/bin/bash
# bench lines of every config (no CPU baseline) — quick A/B after a library-wide change
mkdir -p gpurun_out/ab
for c in ${CONFIGS:-c3 c2 c1 c4 c5}; do
  python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab/all_$c.json 2> gpurun_out/ab/all_$c.err
  echo "$c rc=$?"; python - <<PY
import json
d=json.load(open("gpurun_out/ab/all_$c.json"))
print("  ms/step", d["ms_per_step"], "kernel_us", d["roofline"].get("kernel_us"), "frac", d["roofline"]["frac"])
PY
done
