# Performance ablations of the segmented adjoint phase B and the cached GN scatter (not a product build): PGET_ABLATE=1 removes
# the sweep-B scatter read-modify-writes, 2 the per-band flush, 3 the whole sweep-B walk, 4 the cached
# scatter's HBM entry stream (timing only); 0 = real kernel.
set -x
for a in ${ABL:-1 2 3 0}; do
  PGET_NVCC_EXTRA="-DPGET_ABLATE=$a" python -c "from paper_2604_26745_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  echo "ABLATE=$a"; for c in ${CFGS:-2 4}; do timeout 300 python scripts/time_ops.py $c 20 ${LM:-}; done
done
