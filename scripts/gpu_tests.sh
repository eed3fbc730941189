# GPU test pass (gpurun): pytest -m gpu with durations; log to gpurun_out/
set -x
nproc
timeout 1500 python -m pytest tests -m gpu -q --durations=15 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "^E  .*(Assert|assert )|passed|failed|^[0-9.]+s call" gpurun_out/pytest_gpu.log | head -60
