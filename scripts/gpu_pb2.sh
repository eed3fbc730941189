set -x
timeout 600 python scripts/pb_margin.py > gpurun_out/pb_margin.txt 2>&1
for c in 2 3 4; do timeout 300 python scripts/time_ops.py $c 10 --lm --pb; done > gpurun_out/time_pb.txt 2>&1
for c in 2 4; do timeout 300 python scripts/time_ops.py $c 10 --lm --pb --var; timeout 300 python scripts/time_ops.py $c 10 --lm --var; done >> gpurun_out/time_pb.txt 2>&1
cat gpurun_out/pb_margin.txt gpurun_out/time_pb.txt
