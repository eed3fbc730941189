# cached scatter: b = high-word column address, new = b + exit-test-free 4-sample rounds; bitwise check vs HEAD, A/B, tests
for v in old new; do cp abvar/$v/libpget.so paper_2604_26745_b200/libpget.so && touch paper_2604_26745_b200/libpget.so; python scripts/adj_bitwise.py save $v; done
python scripts/adj_bitwise.py cmp old new | grep -c "bitwise equal"
python scripts/adj_bitwise.py cmp old new | grep DIFFER
bash scripts/ab.sh "old b new" "2 4" --lm > gpurun_out/ab_r2gg.txt 2>&1
cat gpurun_out/ab_r2gg.txt
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "gn_apply or stride or comb or deterministic or cg_loop or lm_iteration" > gpurun_out/pytest_r2gg.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_r2gg.log
