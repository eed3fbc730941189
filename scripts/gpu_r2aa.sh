# A/B: persisting L2 window over the LM iteration's slot partials (PGET_L2_PERSIST=0/1); LM tests incl. graph capture
for r in 1 2; do for v in 0 1; do for c in 2 4 5; do
  echo -n "[l2p $v r$r] "; PGET_L2_PERSIST=$v timeout 600 python scripts/time_ops.py $c 5 --lm 2>&1 | tail -1
done; done; done > gpurun_out/ab_r2aa.txt 2>&1
cat gpurun_out/ab_r2aa.txt
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lm_solve.py -m gpu -q -x -k "lm or graph or cg or solve" > gpurun_out/pytest_r2aa.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_r2aa.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-per-config --no-cpu-baseline > gpurun_out/bench_l2p1.json 2>/dev/null; echo "bench1 rc=$?"
PGET_L2_PERSIST=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-per-config --no-cpu-baseline > gpurun_out/bench_l2p0.json 2>/dev/null; echo "bench0 rc=$?"
python -c "
import json
for f in ('gpurun_out/bench_l2p0.json','gpurun_out/bench_l2p1.json'):
    d=json.load(open(f)); print(f, d['value'], d['ms_per_step'], d['per_op']['lm_ms'], d['roofline']['launch_ms'])"
