# Round profiling bundle (one gpurun call): plain bench, ncu launch list of the bench command,
# ncu --set full of the four projector modes on config 2.  Outputs under gpurun_out/.
set -x
tag=${1:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_$tag.txt
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?"
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_small_$tag.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches_$tag.log 2>&1
echo "ncu launches rc=$?"
timeout 300 python scripts/prof_ops.py 2 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"proj_kernel|seg_|lin_kernel|gnb_kernel" -c 8 \
    -o gpurun_out/full_$tag python scripts/prof_ops.py 2 1 > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu full rc=$?"
