# segmented phase A launch shape: warps per CTA x CTAs per SM
for wc in "8 2" "16 1" "4 4" "12 1" "8 1"; do set -- $wc; echo "SEGA_W=$1 CPS=$2"
  for c in ${CFGS:-2 4}; do PGET_SEGA_W=$1 PGET_SEGA_CPS=$2 timeout 300 python scripts/time_ops.py $c 20; done; done
