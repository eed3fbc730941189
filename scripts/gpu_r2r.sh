# A/B: old = HEAD, b = unrolled sweep-B (VJP) and cache builder, bg = b + keep-FMA pending sums in the cached scatter
bash scripts/ab.sh "old b bg" "2 4" --lm > gpurun_out/ab_r2r.txt 2>&1
cat gpurun_out/ab_r2r.txt
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "stride or gn_apply or lm_iteration or deterministic or config_fwd" > gpurun_out/pytest_r2r.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_r2r.log
