# A/B: 32-bit index arithmetic in the CG vector kernels (new) vs HEAD (old)
bash scripts/ab.sh "old new" "2 4" --lm > gpurun_out/ab_r2y.txt 2>&1
cat gpurun_out/ab_r2y.txt
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lm_solve.py tests/test_gpu_prior.py -m gpu -q -x -k "lm or prior or cg" > gpurun_out/pytest_r2y.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_r2y.log
