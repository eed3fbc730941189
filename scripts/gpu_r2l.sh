# A/B of the branch-free walker loads (old = -DPGET_WALKA_OLD), then the full GPU suite on "new"
bash scripts/ab.sh "old new" "2 4" --lm > gpurun_out/ab_r2l.txt 2>&1
cat gpurun_out/ab_r2l.txt
timeout 2400 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/pytest_r2l.log 2>&1; echo "pytest rc=$?"
tail -12 gpurun_out/pytest_r2l.log
