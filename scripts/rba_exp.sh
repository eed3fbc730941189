# segmented phase A: band-height cap (PGET_RBA_CAP) x segment count (PGET_SEG_K)
for cap in ${CAPS:-32 64}; do for k in ${KS:-0 2 3}; do echo "RBA_CAP=$cap SEG_K=$k"
  for c in ${CFGS:-2 4}; do PGET_RBA_CAP=$cap PGET_SEG_K=$k timeout 300 python scripts/time_ops.py $c 20; done; done; done
