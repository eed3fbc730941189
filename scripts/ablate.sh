# Performance ablations of the projector (not a product build): time each op with the sweep-B
# scatter removed (PGET_ABLATE=1) vs the real kernel (0).
set -x
for a in 1 0; do
  PGET_NVCC_EXTRA="-DPGET_ABLATE=$a" python -c "from paper_2604_26745_b200 import _build; _build.build(force=True)"
  echo "ABLATE=$a"; timeout 300 python scripts/time_ops.py 2 20; timeout 300 python scripts/time_ops.py 3 10
done
