# ncu evidence per config (round 2): launch list of the config-4 bench command, and --set full of one
# launch of each projector kernel on configs 3, 4 and 5.  Outputs under gpurun_out/.
set -x
tag=${1:-r02c}
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-per-config > gpurun_out/bench_small_$tag.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-per-config > gpurun_out/ncu_launches_$tag.log 2>&1
echo "ncu launches rc=$?"
for c in 3 4 5; do
  timeout 300 python scripts/prof_ops.py $c 1 > gpurun_out/prof_plain_$c.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"proj_kernel|seg_|lin_kernel|gnb_kernel" -c 8 \
      -o gpurun_out/full_${tag}_c$c python scripts/prof_ops.py $c 1 > gpurun_out/ncu_full_${tag}_c$c.log 2>&1
  echo "ncu full c$c rc=$?"
done
ls -la gpurun_out/
