# full GPU check: every -m gpu test, the bench line, op timings on all configs
set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json
for c in 1 2 3 4 5; do timeout 300 python scripts/time_ops.py $c 20; done 2>&1 | tee gpurun_out/time_ops_all.log
