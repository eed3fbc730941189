# two phase-A stages (HEAD): band-height cap 64 (default) vs 96 vs 128 on configs 2, 3; then the full state check
set -x
for cap in 64 96 128; do for c in 2 3 4; do echo -n "[cap $cap] "; PGET_RBA_CAP=$cap timeout 300 python scripts/time_ops.py $c 10 --lm 2>&1 | tail -1; done; done | tee gpurun_out/ab_r02oo_rbacap.txt
bash scripts/gpu_r2k.sh r02m
