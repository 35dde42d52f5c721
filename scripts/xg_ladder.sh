#!/bin/bash
# Config-2 hi|lo GEMM timing ladder (timing build): which of loads / MMAs / TMEM reads / y stores
# paces the kernel. Outputs are wrong with any switch set. DEEPTHIN_DBG_XG bits: 1 no y stores
# (st.global epilogue only), 2 no MMAs, 4 no TMEM reads, 8 no dual-A (W_lo) loads.
set -u
mkdir -p gpurun_out/xg
L=$PWD/paper_1802_06944_b200/_lib/libdeepthin_b200_timing.so
for d in ${LADDER:-0 8 2 10}; do
  DEEPTHIN_LIB=$L DEEPTHIN_DBG_XG=$d python bench.py --config c2 --steps 50 --warmup 10 --no-cpu-baseline \
    > gpurun_out/xg/c2_dbg$d.json 2> gpurun_out/xg/c2_dbg$d.err
  echo "dbg=$d rc=$? $(python - <<PY
import json
try:
    j=json.load(open('gpurun_out/xg/c2_dbg$d.json'))
    print(j['ms_per_step'], j['roofline'].get('kernel_us'), j['roofline'].get('kernel_us_raw'))
except Exception as e: print('ERR', e)
PY
)"
done
