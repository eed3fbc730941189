# ncu --set full with source of the eight projector launches of prof_ops.py on config 4 (HEAD)
set -x
tag=${1:-r02j}
timeout 300 python scripts/prof_ops.py 4 1 > gpurun_out/prof_plain_$tag.log 2>&1; echo "plain rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"seg_|lin_kernel|gnb_kernel" -c 8 \
    -o gpurun_out/full_$tag python scripts/prof_ops.py 4 1 > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full_$tag.log
