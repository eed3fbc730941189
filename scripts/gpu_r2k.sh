# round-2 state check r02k (walk_a byte-addressed loads): every -m gpu test, smoke, the bench line, op timings on all
# configs, the ncu launch list of the config-4 bench step and --set full of the projector kernels
set -x
tag=${1:-r02k}
timeout 1500 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/pytest_gpu_$tag.txt 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_$tag.txt
timeout 300 python -c "import __graft_entry__ as G; G.smoke()" > gpurun_out/smoke_$tag.txt 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_$tag.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?"
for c in 1 2 3 4 5; do timeout 300 python scripts/time_ops.py $c 10 --lm; done > gpurun_out/time_ops_$tag.txt 2>&1
cat gpurun_out/time_ops_$tag.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-per-config > gpurun_out/ncu_launches_$tag.log 2>&1
echo "ncu launches rc=$?"
timeout 300 python scripts/prof_ops.py 4 1 > gpurun_out/prof_plain_$tag.log 2>&1; echo "plain rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"proj_kernel|seg_|lin_kernel|gnb_kernel" -c 8 \
    -o gpurun_out/full_$tag python scripts/prof_ops.py 4 1 > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full_$tag.log
