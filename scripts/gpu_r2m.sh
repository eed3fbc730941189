# A/B of the (lam, dlam, mu, dmu) float4 layout with packed GN-mode sums, then the full GPU suite on "new"
bash scripts/ab.sh "old new" "2 4" --lm > gpurun_out/ab_r2m.txt 2>&1
cat gpurun_out/ab_r2m.txt
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_r2m.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_r2m.log
