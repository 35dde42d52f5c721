# usage: bash scripts/gpu_tests.sh [pytest -k expr]
mkdir -p gpurun_out
K=${1:-}
if [ -n "$K" ]; then
  timeout -s KILL 600 python -m pytest tests -m gpu -q --tb=line -rf -k "$K" > gpurun_out/tests.log 2>&1; echo "tests rc=$?"
else
  timeout -s KILL 600 python -m pytest tests -m gpu -q --tb=line -rf > gpurun_out/tests.log 2>&1; echo "tests rc=$?"
fi
tail -45 gpurun_out/tests.log
