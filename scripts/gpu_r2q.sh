# A/B of the unrolled sweep-B walker (old = -DPGET_WALKB_OLD), then the adjoint parity tests on "new"
bash scripts/ab.sh "old new" "2 4 5" --lm > gpurun_out/ab_r2q.txt 2>&1
cat gpurun_out/ab_r2q.txt
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variant.py -m gpu -q -x > gpurun_out/pytest_r2q.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_r2q.log
