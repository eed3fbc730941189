# reduction blocks per member (kNblk) 64 vs 128 vs 148: A/B on the LM iteration
set -x
cp paper_2604_26745_b200/libpget.so /tmp/new.so
bash scripts/ab.sh "bs nb128 nb148" "2 4 5" --lm 2>&1 | tee gpurun_out/ab_r02mm_nblk.txt
cp /tmp/new.so paper_2604_26745_b200/libpget.so
