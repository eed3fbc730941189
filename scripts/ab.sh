# A/B timing of library variants: abvar/<name>/libpget.so, each installed in turn (touched newer
# than the sources so the binding does not rebuild), then time_ops on the configs in $CFGS.
# usage: bash scripts/ab.sh "old new" "2 3 4" [time_ops flags]
vars=$1; cfgs=${2:-"2 4"}; shift 2
for r in 1 2; do
for v in $vars; do
  cp abvar/$v/libpget.so paper_2604_26745_b200/libpget.so && touch paper_2604_26745_b200/libpget.so
  for c in $cfgs; do echo -n "[$v r$r] "; timeout 300 python scripts/time_ops.py $c 10 "$@" 2>&1 | tail -1; done
done
done
