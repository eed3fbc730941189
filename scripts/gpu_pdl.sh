set -x
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_g.log 2>&1; echo "pytest rc=$?"
grep -E "^E  .*(Assert|assert )|passed|failed" gpurun_out/pytest_g.log | head -20
for p in 1 0; do echo "== PGET_PDL=$p"; for c in 1 2 4; do PGET_PDL=$p timeout 300 python scripts/time_ops.py $c 10 --lm; done; done > gpurun_out/pdl.txt 2>&1
cat gpurun_out/pdl.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_g.json 2> gpurun_out/bench_g.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench_g.json
