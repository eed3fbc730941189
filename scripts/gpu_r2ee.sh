# the cached scatter with the fraction offsets folded into FMAs: bitwise check (VJP, GN apply, LM iteration) and A/B
for v in old new; do cp abvar/$v/libpget.so paper_2604_26745_b200/libpget.so && touch paper_2604_26745_b200/libpget.so; python scripts/adj_bitwise.py save $v; done
python scripts/adj_bitwise.py cmp old new
bash scripts/ab.sh "old new" "2 4" --lm > gpurun_out/ab_r2ee.txt 2>&1
cat gpurun_out/ab_r2ee.txt
