# phase-A stage buffers (PGET_SEGA_STAGES)
for n in ${NS:-2 4 3}; do
  PGET_NVCC_EXTRA="-DPGET_SEGA_STAGES=$n" python -c "from paper_2604_26745_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  echo "STAGES=$n"; for c in 2 4; do timeout 300 python scripts/time_ops.py $c 10 --lm; done
done
