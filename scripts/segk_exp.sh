# segmented adjoint: segment count sweep (PGET_SEG_K) and the per-kernel split of one GN product
for k in ${KS:-1 2 3 4}; do echo "SEG_K=$k"; for c in ${CFGS:-2 3 4}; do PGET_SEG_K=$k timeout 300 python scripts/time_ops.py $c 20; done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"seg_|reduce|finish|pack" python scripts/prof_ops.py 2 1 > gpurun_out/seg_launches.csv 2>/dev/null
grep -E "seg_|reduce_slots" gpurun_out/seg_launches.csv | awk -F'","' '{print $5, $NF}' | head -20
