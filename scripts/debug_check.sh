# Bounds-checked build (-DPGET_DEBUG: __trap on any out-of-range shared-memory index in the sample
# loops) run through the small and edge-case parity tests, then the normal build is restored.
set -x
PGET_NVCC_EXTRA="-DPGET_DEBUG" python -c "from paper_2604_26745_b200 import _build; _build.build(force=True)"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x \
    -k "edge_geometries or degenerate or errors_fail or small_batched or config_fwd_jvp_vjp or gn_apply or lm_iteration_cfg2" > gpurun_out/debug_check.log 2>&1
echo "debug tests rc=$?"; tail -3 gpurun_out/debug_check.log
python -c "from paper_2604_26745_b200 import _build; _build.build(force=True)"
