# A/B: the fused CG kernel launched cooperative + PDL (PGET_CG_PDL=1) vs plain cooperative; LM tests and graph capture
for r in 1 2; do for v in 0 1; do for c in 1 2 4; do
  echo -n "[cgpdl $v r$r] "; PGET_CG_PDL=$v timeout 600 python scripts/time_ops.py $c 10 --lm 2>&1 | tail -1
done; done; done > gpurun_out/ab_r2bb.txt 2>&1
cat gpurun_out/ab_r2bb.txt
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lm_solve.py -m gpu -q -x -k "lm or graph or cg or solve or batched" > gpurun_out/pytest_r2bb.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_r2bb.log
