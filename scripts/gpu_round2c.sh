# variant parity, gnb experiment variants (PGET_GNB_MODE 0-3), shared atomics micro
set -x
timeout 900 python -m pytest tests/test_gpu_variant.py -q -x > gpurun_out/variant.log 2>&1; echo "variant rc=$?"
grep -E "^E  .*(Assert)|passed|failed" gpurun_out/variant.log | head
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/smem_atom scripts/micro/smem_atom.cu && /tmp/smem_atom > gpurun_out/smem_atom.txt 2>&1; cat gpurun_out/smem_atom.txt
for m in 0 1 2 3; do
  PGET_NVCC_EXTRA="-DPGET_GNB_MODE=$m" python -c "import sys; sys.path.insert(0,'paper_2604_26745_b200'); import _build; _build.build(force=True)" > /dev/null 2>&1
  echo "== mode $m"
  for c in 2 4; do timeout 300 python scripts/time_ops.py $c 10 --lm; done
  PGET_GN_APPLY_CACHED=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "gn_apply_operator and cached and not float" 2>&1 | tail -1
done > gpurun_out/gnb_modes.txt 2>&1
cat gpurun_out/gnb_modes.txt
