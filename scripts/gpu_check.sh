set -x
timeout 900 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "^E  .*(Assert|assert )|passed|failed" gpurun_out/pytest_gpu.log | head -30
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d['per_op'])); print(d['value'], d['roofline']['frac'])"
