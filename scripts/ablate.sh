# Performance ablations of the projector (not a product build): PGET_ABLATE=1 removes the sweep-B
# scatter, 2 the per-band ring flush, 3 every sweep-B walk, 4 every sweep-A walk; 0 is the real kernel.
set -x
for a in ${ABL:-1 2 0}; do
  PGET_NVCC_EXTRA="-DPGET_ABLATE=$a" python -c "from paper_2604_26745_b200 import _build; _build.build(force=True)"
  echo "ABLATE=$a"; timeout 300 python scripts/time_ops.py 2 20; timeout 300 python scripts/time_ops.py 4 5
done
