# run the phase trace with alternative builds of the library (scripts/variants/lib_*.so)
cp paper_1802_06944_b200/_lib/libdeepthin_b200.so /tmp/orig.so
for v in scripts/variants/lib_*.so; do
  cp $v paper_1802_06944_b200/_lib/libdeepthin_b200.so
  echo "== $v"
  DEEPTHIN_TC_TRACE=1 timeout 60 python scripts/prof_forward.py --iters 3 > gpurun_out/tr.log 2>&1
  grep -E "span|cta  63" -A1 gpurun_out/tr.log | tail -3
done
cp /tmp/orig.so paper_1802_06944_b200/_lib/libdeepthin_b200.so
