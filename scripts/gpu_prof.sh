set -x
tag=${1:-x}
timeout 300 python scripts/prof_ops.py 2 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:proj_kernel -c 4 -o gpurun_out/prof_$tag python scripts/prof_ops.py 2 1 > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_full.log
