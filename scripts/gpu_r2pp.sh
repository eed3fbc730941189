# cached scatter's entry loads with an L2 evict-first policy (PGET_GNB_EF=1) vs HEAD: A/B on the LM iteration
set -x
cp paper_2604_26745_b200/libpget.so /tmp/new.so
bash scripts/ab.sh "head ef" "2 4 5" --lm 2>&1 | tee gpurun_out/ab_r02pp_ef.txt
cp /tmp/new.so paper_2604_26745_b200/libpget.so
