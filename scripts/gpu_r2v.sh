# ablations of the cached scatter inside the LM iteration (1: no scatter, 2: no flush, 3: no walk)
ABL="1 2 3 0" CFGS="2 4" LM="--lm" bash scripts/ablate.sh > gpurun_out/ablate_r2v.txt 2>&1
grep -v "^+" gpurun_out/ablate_r2v.txt
