#!/bin/bash
# A/B of the two row kernels on config 3 (bench lines only)
mkdir -p gpurun_out/ab
for k in 1 0; do
  DEEPTHIN_ROWS_SLAB=$k python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab/c3_slab$k.json 2> gpurun_out/ab/c3_slab$k.err
  echo "slab=$k rc=$?"; python - <<PY
import json
d=json.load(open("gpurun_out/ab/c3_slab$k.json"))
print(d["ms_per_step"], d["roofline"]["kernel_us"], d["roofline"]["frac"], d["roofline"].get("kernel"))
PY
done
