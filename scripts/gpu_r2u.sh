# sparse per-warp flush of sweep B (old = -DPGET_DENSE_FLUSH): bitwise check, A/B, adjoint parity tests
for v in old new; do cp abvar/$v/libpget.so paper_2604_26745_b200/libpget.so && touch paper_2604_26745_b200/libpget.so; python scripts/adj_bitwise.py save $v; done
python scripts/adj_bitwise.py cmp old new
bash scripts/ab.sh "old new" "2 4" > gpurun_out/ab_r2u.txt 2>&1
cat gpurun_out/ab_r2u.txt
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "config_fwd or deterministic or gn_apply or high_optical or edge or adjoint" > gpurun_out/pytest_r2u.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_r2u.log
