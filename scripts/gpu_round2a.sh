# stress test + bench (config 4, per-config) + LDS peak + ncu launch list of the bench step
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/smem_bw scripts/micro/smem_bw.cu && /tmp/smem_bw > gpurun_out/smem_bw.txt 2>&1
cat gpurun_out/smem_bw.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k high_optical > gpurun_out/stress.log 2>&1; echo "stress rc=$?"
grep -E "^E  .*(Assert|assert |rel_l2)|passed|failed" gpurun_out/stress.log | head -20
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_c4.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-per-config > gpurun_out/ncu_c4.log 2>&1; echo "ncu rc=$?"
