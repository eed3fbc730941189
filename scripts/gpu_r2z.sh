# ncu --set full of the projector kernels on config 5 (the batched, HBM-bound case) at HEAD
timeout 300 python scripts/prof_ops.py 5 1 > gpurun_out/prof_plain_c5.log 2>&1; echo "plain rc=$?"
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"seg_|lin_kernel|gnb_kernel" -c 8 \
    -o gpurun_out/full_r02h_c5 python scripts/prof_ops.py 5 1 > gpurun_out/ncu_full_c5.log 2>&1
echo "ncu full rc=$?"
