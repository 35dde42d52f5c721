#!/bin/bash
# Config-2 A/B (timing build): stage count / TMA-store epilogue / regen co-residency.
set -u
mkdir -p gpurun_out/xg
L=$PWD/paper_1802_06944_b200/_lib/libdeepthin_b200_timing.so
run() {  # name, env...
  local name=$1; shift
  env DEEPTHIN_LIB=$L "$@" python bench.py --config c2 --steps 50 --warmup 10 --no-cpu-baseline \
    > gpurun_out/xg/ab_$name.json 2> gpurun_out/xg/ab_$name.err
  echo "$name rc=$? $(python - <<PY
import json
try:
    j=json.load(open('gpurun_out/xg/ab_$name.json'))
    print(j['ms_per_step'], j['roofline'].get('kernel_us'), j['roofline'].get('kernel_us_raw'))
except Exception as e: print('ERR', e)
PY
)"
}
run default A=1
run s4 DEEPTHIN_DBG_XG_S=4
run s3_notma DEEPTHIN_DBG_XG_NOTMA=1
run s4_notma DEEPTHIN_DBG_XG_NOTMA=1 DEEPTHIN_DBG_XG_S=4
run s2 DEEPTHIN_DBG_XG_S=2
