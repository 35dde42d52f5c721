# Round-1 evidence pass: GPU tests, bench lines for configs 2-5, ncu launch lists and one
# --set full capture of the row-tile kernel (each ncu run only after its command exits 0).
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q --tb=line -rf > gpurun_out/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/tests.log
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
for c in c2 c3 c4 c5; do python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"; done
python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c3.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_bench_launches.csv \
      python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1; echo "ncu c3 launches rc=$?"
python scripts/c3_probe.py > gpurun_out/plain_probe.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_tc_rows -s 2 -c 1 \
      -o gpurun_out/prof_rows python scripts/c3_probe.py > gpurun_out/ncu_rows.log 2>&1; echo "ncu full rows rc=$?"
