#!/bin/bash
# env sweep of the clustered row-tile kernel on config 3
mkdir -p gpurun_out/ab
run() {
  env "$@" python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab/sw.json 2> gpurun_out/ab/sw.err
  python - "$*" <<PY
import json,sys
d=json.load(open("gpurun_out/ab/sw.json"))
print(sys.argv[1], "->", d["ms_per_step"], d["roofline"]["kernel_us"], d["roofline"]["frac"])
PY
}
run DEEPTHIN_ROWS_SLAB=0
run DEEPTHIN_ROWS_SLAB=0 DEEPTHIN_ROWS_ND=3
run DEEPTHIN_ROWS_SLAB=0 DEEPTHIN_ROWS_STG=2
run DEEPTHIN_ROWS_SLAB=0 DEEPTHIN_ROWS_ND=3 DEEPTHIN_ROWS_STG=2
run DEEPTHIN_ROWS_SLAB=0 DEEPTHIN_ROWS_CS=8
run DEEPTHIN_ROWS_SLAB=0 DEEPTHIN_ROWS_CS=2
run DEEPTHIN_ROWS_SLAB=1 DEEPTHIN_SLAB_BS=3
run DEEPTHIN_ROWS_SLAB=1 DEEPTHIN_SLAB_STG=2
run DEEPTHIN_ROWS_SLAB=1 DEEPTHIN_SLAB_CTAS=132
