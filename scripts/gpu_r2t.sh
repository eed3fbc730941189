# batched LM tests with the interleaved cache layout for batches; sweep-B ablations (1: no scatter, 2: no flush, 3: no walk)
timeout 1800 python -m pytest tests -m gpu -q -x -k "batched or config5 or lm_solve or prior or safeguard" > gpurun_out/pytest_r2t.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_r2t.log
ABL="1 2 3 0" CFGS="2 4" bash scripts/ablate.sh > gpurun_out/ablate_r2t.txt 2>&1
grep -v "^+" gpurun_out/ablate_r2t.txt
