for d in ${DS:-4 8 12}; do
  X="-DPGET_PF_DIST=$d"   # <= 12: the read-ahead stays inside the cache's padding rows
  PGET_NVCC_EXTRA="$X" python -c "from paper_2604_26745_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  echo "PF=$d"; for c in 2 4; do timeout 300 python scripts/time_ops.py $c 10 --lm; done
done
