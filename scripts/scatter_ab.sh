# A/B of the sweep-B scatter variants (PGET_SCATTER 1 = pending-cell registers, 0 = per-sample RMW)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gn_apply or config_fwd or edge or determin or degenerate or adjoint_identity" > gpurun_out/sc_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/sc_pytest.log
for c in 2 3 4; do timeout 300 python scripts/time_ops.py $c 20; done
PGET_NVCC_EXTRA="-DPGET_SCATTER=0" python -c "from paper_2604_26745_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
echo "SCATTER=0"
for c in 2 3 4; do timeout 300 python scripts/time_ops.py $c 20; done
