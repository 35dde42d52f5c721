# One GPU session: tests, smoke, bench, reference arm, ncu launch list + full captures of the
# two forward kernels (phase-1 W^T regeneration, phase-2 tcgen05 GEMM).
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q --tb=line -rf > gpurun_out/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/tests.log
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.json
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python scripts/prof_forward.py > gpurun_out/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm -c 1 \
      -o gpurun_out/prof_gemm python scripts/prof_forward.py > gpurun_out/ncu_full.log 2>&1; echo "ncu full gemm rc=$?"
python scripts/prof_forward.py > gpurun_out/plain3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_regen_wt -c 1 \
      -o gpurun_out/prof_regen python scripts/prof_forward.py > gpurun_out/ncu_full2.log 2>&1; echo "ncu full regen rc=$?"
