# ncu evidence per config (round 2): launch list of the config-4 bench command, and --set full of one
# launch of each projector kernel on configs 3, 4 and 5, summarised ON the box (the .ncu-rep files are
# too large to bring back): gpurun_out/prof_<tag>/ gets the summaries, launch list and raw csv pages.
set -x
tag=${1:-r02c}
out=gpurun_out/prof_$tag
mkdir -p $out
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-per-config > $out/bench_small.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-per-config > $out/ncu_launches.log 2>&1
echo "ncu launches rc=$?"
for c in ${CFGS:-3 4 5}; do
  timeout 300 python scripts/prof_ops.py $c 1 > $out/prof_plain_$c.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"proj_kernel|seg_|lin_kernel|gnb_kernel" -c 8 \
      -o /tmp/full_${tag}_c$c python scripts/prof_ops.py $c 1 > $out/ncu_full_c$c.log 2>&1
  echo "ncu full c$c rc=$?"
  python scripts/ncu_summary.py ${tag}_c$c $out/launches.csv /tmp/full_${tag}_c$c.ncu-rep $c > /dev/null 2>&1
  cp profiles/ncu_summary_${tag}_c$c.md $out/
  ncu -i /tmp/full_${tag}_c$c.ncu-rep --page source --csv > $out/source_c$c.csv 2>/dev/null
  gzip -f $out/source_c$c.csv
done
cp profiles/ncu_sol.json profiles/traffic.json $out/ 2>/dev/null
du -sh $out
