# Performance ablations of the projector (not a product build): PGET_ABLATE=1 removes the sweep-B
# scatter, 2 removes the per-band ring flush; 0 is the real kernel.
set -x
for a in 2 1 0; do
  PGET_NVCC_EXTRA="-DPGET_ABLATE=$a" python -c "from paper_2604_26745_b200 import _build; _build.build(force=True)"
  echo "ABLATE=$a"; timeout 300 python scripts/time_ops.py 2 20; timeout 300 python scripts/time_ops.py 4 5
done
