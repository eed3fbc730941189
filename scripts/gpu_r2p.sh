# A/B: segments per angle-bank (PGET_SEG_K) on configs 2-4, LM iteration and GN product
for r in 1 2; do for k in 0 1 2 3 4; do for c in 2 3 4; do
  echo -n "[K $k r$r] "; if [ $k = 0 ]; then timeout 300 python scripts/time_ops.py $c 10 --lm 2>&1 | tail -1;
  else PGET_SEG_K=$k timeout 300 python scripts/time_ops.py $c 10 --lm 2>&1 | tail -1; fi
done; done; done > gpurun_out/ab_r2p.txt 2>&1
cat gpurun_out/ab_r2p.txt
