set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variant.py -m gpu -q -x -k "config_fwd or gn_apply_operator or cg_loop or lm_iteration or high_optical or variant_fwd" > gpurun_out/pytest_sw.log 2>&1; echo "pytest rc=$?"
grep -E "^E  .*(Assert|assert )|passed|failed" gpurun_out/pytest_sw.log | head -20
for w in 1 0; do echo "== PGET_SEGA_WIDE=$w"; for c in 3 4; do PGET_SEGA_WIDE=$w timeout 300 python scripts/time_ops.py $c 10 --lm; done; done > gpurun_out/sega2.txt 2>&1
cat gpurun_out/sega2.txt
