# full GPU suite, smoke, default bench (config 4), per-config op timings
set -x
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu_i.log 2>&1; echo "pytest rc=$?"
grep -E "^E  .*(Assert|assert )|passed|failed" gpurun_out/pytest_gpu_i.log | head -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_i.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_i.json 2> gpurun_out/bench_i.err; echo "bench rc=$?"
for c in 1 2 3 4 5; do timeout 300 python scripts/time_ops.py $c 10 --lm; done > gpurun_out/time_ops_i.txt 2>&1
cat gpurun_out/time_ops_i.txt
