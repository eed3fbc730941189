set -x
timeout 900 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "^E  .*(Assert|assert )|passed|failed" gpurun_out/pytest_gpu.log | head -30
timeout 300 python scripts/prof_ops.py 2 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:proj_kernel -c 4 -o gpurun_out/prof_r1b_cfg2 python scripts/prof_ops.py 2 1 > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_full.log
