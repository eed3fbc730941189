set -x
timeout 900 python -m pytest tests/test_gpu_pixel_basis.py -q -x --durations=8 > gpurun_out/pytest_pb.log 2>&1; echo "pytest rc=$?"
grep -E "^E  |passed|failed|Error" gpurun_out/pytest_pb.log | head -30
