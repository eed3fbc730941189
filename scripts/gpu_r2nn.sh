# phase-A stage buffers 3 (HEAD) vs 2 (taller bands) vs 4: A/B
set -x
cp paper_2604_26745_b200/libpget.so /tmp/new.so
bash scripts/ab.sh "bs st2 st4" "2 4" --lm 2>&1 | tee gpurun_out/ab_r02nn_stages.txt
cp /tmp/new.so paper_2604_26745_b200/libpget.so
