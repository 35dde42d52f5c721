#!/bin/bash
# both row kernels at the per-GPU shard sizes of 2/4/8-GPU jobs (config 3, one GPU)
mkdir -p gpurun_out/ab
for n in 1 2 4 8; do for k in 0 1; do
  DEEPTHIN_ROWS_SLAB=$k python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline --shard-of $n > gpurun_out/ab/sh.json 2> gpurun_out/ab/sh.err
  python - $n $k <<PY
import json,sys
d=json.load(open("gpurun_out/ab/sh.json"))
print("shard-of", sys.argv[1], "slab", sys.argv[2], "batch", d["config"]["batch_per_gpu"], "->", d["ms_per_step"]*1e3, "us; rows kernel", d["roofline"]["kernel_us"])
PY
done; done
