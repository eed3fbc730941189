# full GPU suite (rebased paired sums, variant, pairing flag), stress, gnb timing ablations
set -x
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu_d.log 2>&1; echo "pytest rc=$?"
grep -E "^E  .*(Assert|assert )|passed|failed" gpurun_out/pytest_gpu_d.log | head -30
cp paper_2604_26745_b200/libpget.so /tmp/libpget_default.so
for m in "PGET_GNB_MODE=4" "PGET_GNB_MODE=8" "PGET_ABLATE=1"; do
  PGET_NVCC_EXTRA="-D$m" python -c "import sys; sys.path.insert(0,'paper_2604_26745_b200'); import _build; _build.build(force=True)" > /dev/null 2>&1
  echo "== $m"
  for c in 2 4; do timeout 300 python scripts/time_ops.py $c 10 --lm; done
done > gpurun_out/gnb_abl.txt 2>&1
cat gpurun_out/gnb_abl.txt
cp /tmp/libpget_default.so paper_2604_26745_b200/libpget.so
for c in 2 4; do timeout 300 python scripts/time_ops.py $c 10 --lm; done
