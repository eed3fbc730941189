# quick GPU check after a kernel change: the parity subset most sensitive to projector changes + timings
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gn_apply or config_fwd or edge or determin or lm_iteration" > gpurun_out/quick_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/quick_pytest.log
for c in ${QC_CONFIGS:-2 4}; do timeout 300 python scripts/time_ops.py $c 20 ${QC_LM:-}; done 2>&1 | tee gpurun_out/quick_time.log
