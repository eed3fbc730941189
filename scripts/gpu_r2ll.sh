# band_steps by an fp32 estimate + exact fix-up: parity subset, then A/B lds (HEAD) vs bs
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gn_apply or config_fwd or edge or determin or lm_iteration or high_optical or degenerate" > gpurun_out/quick_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/quick_pytest.log
cp paper_2604_26745_b200/libpget.so /tmp/new.so
bash scripts/ab.sh "lds bs" "2 4" --lm 2>&1 | tee gpurun_out/ab_r02ll_bs.txt
cp /tmp/new.so paper_2604_26745_b200/libpget.so
