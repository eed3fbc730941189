# round-end evidence at HEAD: full GPU suite, smoke, bench (config 4), launch list, ncu --set full (config 4), per-config timings
set -x
tag=${1:-r02h}
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_$tag.txt
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err; echo "ref rc=$?"
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-per-config > gpurun_out/bench_small_$tag.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-per-config > gpurun_out/ncu_launches_$tag.log 2>&1
echo "ncu launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"seg_|lin_kernel|gnb_kernel" -c 8 \
    -o gpurun_out/full_$tag python scripts/prof_ops.py 4 1 > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu full rc=$?"
for c in 1 2 3 4 5; do timeout 300 python scripts/time_ops.py $c 10 --lm; done > gpurun_out/time_ops_$tag.txt 2>&1
cat gpurun_out/time_ops_$tag.txt | grep cfg
