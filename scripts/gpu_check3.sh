set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "config_fwd or config5 or edge or degenerate or high_optical or safeguard or variant or gn_apply_operator or cg_loop" > gpurun_out/pytest_f.log 2>&1; echo "pytest rc=$?"
grep -E "^E  .*(Assert|assert )|passed|failed" gpurun_out/pytest_f.log | head -20
for c in 1 2 3 4 5; do timeout 300 python scripts/time_ops.py $c 10 --lm; done > gpurun_out/time_f.txt 2>&1
cat gpurun_out/time_f.txt
