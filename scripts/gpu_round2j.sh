# HEAD state check (round 2, session 5): GPU suite, smoke, default bench (config 4), per-config op
# timings, the bench command's ncu launch list, ncu --set full of the config-4 GN launch pair
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_r02j.txt
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu_r02j.log 2>&1; echo "pytest rc=$?"
grep -E "^E  .*(Assert|assert )|passed|failed" gpurun_out/pytest_gpu_r02j.log | head -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02j.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_r02j.json 2> gpurun_out/bench_r02j.err; echo "bench rc=$?"
for c in 1 2 3 4 5; do timeout 300 python scripts/time_ops.py $c 10 --lm; done > gpurun_out/time_ops_r02j.txt 2>&1
cat gpurun_out/time_ops_r02j.txt
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_small_r02j.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02j.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches_r02j.log 2>&1
echo "ncu launches rc=$?"
timeout 300 python scripts/prof_ops.py 4 1 > gpurun_out/prof_plain_r02j.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"proj_kernel|seg_|lin_kernel|gnb_kernel" -c 8 \
    -o gpurun_out/full_r02j python scripts/prof_ops.py 4 1 > gpurun_out/ncu_full_r02j.log 2>&1
echo "ncu full rc=$?"
