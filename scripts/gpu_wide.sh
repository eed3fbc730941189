set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "gn_apply_operator or cg_loop or lm_iteration" > gpurun_out/pytest_w.log 2>&1; echo "pytest rc=$?"
grep -E "^E  .*(Assert|assert )|passed|failed" gpurun_out/pytest_w.log | head -20
for w in 1 0; do echo "== PGET_GNB_WIDE=$w"; for c in 3 4; do PGET_GNB_WIDE=$w timeout 300 python scripts/time_ops.py $c 10 --lm; done; done > gpurun_out/wide.txt 2>&1
cat gpurun_out/wide.txt
