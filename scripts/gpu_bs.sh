set -x
for m in 1 0; do
  PGET_NVCC_EXTRA="-DPGET_BANDSTEPS=$m" python -c "import sys; sys.path.insert(0,'paper_2604_26745_b200'); import _build; _build.build(force=True)" > /dev/null 2>&1
  echo "== bandsteps $m"
  for c in 2 4 5; do timeout 300 python scripts/time_ops.py $c 10 --lm; done
done > gpurun_out/bs.txt 2>&1
cat gpurun_out/bs.txt
