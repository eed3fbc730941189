# state check after re-entry: full GPU suite, smoke, default bench, per-config op timings
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_e.txt
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu_e.log 2>&1; echo "pytest rc=$?"
grep -E "^E  .*(Assert|assert )|passed|failed" gpurun_out/pytest_gpu_e.log | head -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_e.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err; echo "bench rc=$?"
for c in 1 2 3 4 5; do timeout 300 python scripts/time_ops.py $c 10 --lm; done > gpurun_out/time_ops_e.txt 2>&1
cat gpurun_out/time_ops_e.txt | tail -40
