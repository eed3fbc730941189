# segmented adjoint: parity subset + timings, then the fused adjoint for comparison
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gn_apply or config_fwd or edge or determin or degenerate or adjoint_identity" > gpurun_out/seg_pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/seg_pytest.log
for c in 2 3 4; do timeout 300 python scripts/time_ops.py $c 20; done
for c in 2 3; do PGET_ADJ_FUSED=1 timeout 300 python scripts/time_ops.py $c 20; done
