# gnb_kernel: shared 32-bit fixed-point accumulator (PGET_GNB_INT=1, default) vs per-warp float accumulators (0)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gn_apply or lm_iteration or determin or edge or degenerate" 2>&1 | tail -3
for v in 1 0; do
  echo "GNB_INT=$v"; for c in 2 3 4; do PGET_GNB_INT=$v timeout 300 python scripts/time_ops.py $c 20 --lm; done
done
