set -x
for w in 13 14 15; do echo "== PGET_SEGA_W=$w"; for c in 3 4; do PGET_SEGA_W=$w timeout 300 python scripts/time_ops.py $c 10 --lm; done; done > gpurun_out/sega.txt 2>&1
cat gpurun_out/sega.txt
