# A/B: phase-A CTAs per SM (PGET_SEGA_CPS) on configs 1-4
for r in 1 2; do for cps in 1 2; do for c in 1 2 3 4; do
  echo -n "[cps $cps r$r] "; PGET_SEGA_CPS=$cps timeout 300 python scripts/time_ops.py $c 10 --lm 2>&1 | tail -1
done; done; done > gpurun_out/ab_r2w.txt 2>&1
cat gpurun_out/ab_r2w.txt
