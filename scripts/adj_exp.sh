# cached GN path over consecutive-ray groups (PGET_GNB_ADJ=1) vs comb groups: LM iteration, GN apply
cp abvar/adj/libpget.so paper_2604_26745_b200/libpget.so && touch paper_2604_26745_b200/libpget.so
for r in 1 2; do for a in 0 1; do
  for c in 2 3 4 5; do echo -n "[adj=$a r$r] "; PGET_GNB_ADJ=$a timeout 300 python scripts/time_ops.py $c 6 --lm 2>&1 | tail -1; done
done; done
PGET_GNB_ADJ=1 PGET_GN_APPLY_CACHED=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gn_apply or lm_iteration or cg_loop or determ" 2>&1 | tail -3
