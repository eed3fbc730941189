# final state check at HEAD: full GPU suite, smoke, bench (config 4)
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r02i.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu_r02i.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02i.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_r02i.json 2> gpurun_out/bench_r02i.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/bench_r02i.json'))
print(d['value'],d['ms_per_step'],d['per_op']['lm_ms'],d['roofline']['frac'],d['roofline']['launch_ms'],d['clocks'],d['e2e']['value'])"
