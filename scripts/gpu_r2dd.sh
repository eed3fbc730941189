# ablation 4: the cached scatter without its HBM entry stream (timing only) vs the real kernel, LM configs 2/4/5
ABL="4 0" CFGS="2 4" LM="--lm" bash scripts/ablate.sh > gpurun_out/ablate_r2dd.txt 2>&1
grep -v "^+" gpurun_out/ablate_r2dd.txt
