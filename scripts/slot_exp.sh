# units per fp32 partial slot (PGET_SLOT_TASKS): LM iteration on configs 4 and 5
for st in 16 32 64; do
  echo "== PGET_SLOT_TASKS=$st"
  for c in 4 5; do PGET_SLOT_TASKS=$st timeout 300 python scripts/time_ops.py $c 6 --lm; done
done
