# schedule experiment: detector-range parts capped at PGET_SCHED_PMAX (1 = whole angle-banks)
for pm in ${PMS:-1 2 3}; do echo "PMAX=$pm"; for c in ${CFGS:-2 3 4}; do PGET_SCHED_PMAX=$pm timeout 300 python scripts/time_ops.py $c 20; done; done
