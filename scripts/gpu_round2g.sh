set -x
timeout 900 python -m pytest tests/test_gpu_pixel_basis.py -q -x > gpurun_out/pytest_pb_g.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_pb_g.log
for c in 2 4; do timeout 300 python scripts/time_ops.py $c 10 --lm --pb; done > gpurun_out/time_pb_g.txt 2>&1; cat gpurun_out/time_pb_g.txt
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_g.json 2> gpurun_out/bench_g.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_g.json')); print(d['per_config']['config 5'].get('hbm'))"
