# config 5: the consecutive/interleaved cache layout (PGET_GNB_ADJ=1) vs the comb layout (default for batches);
# config 2: ncu of the GN kernels
for r in 1 2; do
  echo -n "[adj0 r$r] "; timeout 600 python scripts/time_ops.py 5 5 --lm 2>&1 | tail -1
  echo -n "[adj1 r$r] "; PGET_GNB_ADJ=1 timeout 600 python scripts/time_ops.py 5 5 --lm 2>&1 | tail -1
done > gpurun_out/ab_r2s.txt 2>&1
cat gpurun_out/ab_r2s.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"seg_|lin_kernel|gnb_kernel" -c 8 \
    -o gpurun_out/full_r02s_c2 python scripts/prof_ops.py 2 1 > gpurun_out/ncu_full_r02s.log 2>&1; echo "ncu rc=$?"
