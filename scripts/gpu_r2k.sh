# A/B: cached-scatter group stride (PGET_GNB_STRIDE) and the forward-mode phase A (PGET_FWD_PLAIN)
set -x
for r in 1 2; do
for st in 1 2 3 4; do
  for c in 2 4; do echo -n "[stride $st r$r] "; PGET_GNB_STRIDE=$st timeout 300 python scripts/time_ops.py $c 10 --lm 2>&1 | tail -1; done
done
for fp in 0 1; do
  for c in 2 4; do echo -n "[fwdplain $fp r$r] "; PGET_FWD_PLAIN=$fp timeout 300 python scripts/time_ops.py $c 10 2>&1 | tail -1; done
done
done > gpurun_out/ab_r2k.txt 2>&1
cat gpurun_out/ab_r2k.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "forward or lm or gn" > gpurun_out/pytest_r2k.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_r2k.log
