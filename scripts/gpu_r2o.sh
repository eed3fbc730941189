# experiment: the standalone VJP through the coefficient cache (PGET_VJP_CACHED=1) -- parity margins and timing
for v in 0 1; do PGET_VJP_CACHED=$v timeout 900 python scripts/vjp_margin.py 1 2 3 4; done > gpurun_out/vjp_margin_r2o.txt 2>&1
cat gpurun_out/vjp_margin_r2o.txt
for r in 1 2; do for v in 0 1; do for c in 2 4; do echo -n "[vjpc $v r$r] "; PGET_VJP_CACHED=$v timeout 300 python scripts/time_ops.py $c 10 2>&1 | tail -1; done; done; done > gpurun_out/ab_r2o.txt 2>&1
cat gpurun_out/ab_r2o.txt
