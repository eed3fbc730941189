# optical-depth diagnosis (paired vs unpaired), unpaired parity subset, config-4 ncu full capture
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k high_optical > gpurun_out/stress_pair.log 2>&1; echo "stress paired rc=$?"
grep -E "^E  .*(Assert)|passed|failed" gpurun_out/stress_pair.log | head
PGET_NO_PAIR=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k high_optical > gpurun_out/stress_nopair.log 2>&1; echo "stress nopair rc=$?"
grep -E "^E  .*(Assert)|passed|failed" gpurun_out/stress_nopair.log | head
PGET_NO_PAIR=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "config_fwd or gn_apply_operator or lm_iteration or edge or cg_loop" > gpurun_out/nopair.log 2>&1; echo "nopair parity rc=$?"
grep -E "^E  .*(Assert)|passed|failed" gpurun_out/nopair.log | head
for c in 2 4; do PGET_NO_PAIR=1 timeout 300 python scripts/time_ops.py $c 10 --lm; done > gpurun_out/time_nopair.txt 2>&1
cat gpurun_out/time_nopair.txt
timeout 300 python scripts/prof_ops.py 4 1 > gpurun_out/prof_plain4.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"proj_kernel|seg_|lin_kernel|gnb_kernel" -c 8 \
    -o gpurun_out/full_c4 python scripts/prof_ops.py 4 1 > gpurun_out/ncu_full_c4.log 2>&1
echo "ncu full rc=$?"
