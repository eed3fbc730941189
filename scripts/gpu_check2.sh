# parity subset + per-op timings on configs 1-5
set -x
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_e.log 2>&1; echo "pytest rc=$?"
grep -E "^E  .*(Assert|assert )|passed|failed" gpurun_out/pytest_e.log | head -20
for c in 1 2 3 4 5; do timeout 300 python scripts/time_ops.py $c 10 --lm; done > gpurun_out/time_e.txt 2>&1
cat gpurun_out/time_e.txt
