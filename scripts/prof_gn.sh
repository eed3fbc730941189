# ncu --set full of the GN projector kernels on configs 2 and 4 (one launch each; KRE selects them)
set -x
tag=${1:-x}
for c in ${CFGS:-2 4}; do
  timeout 300 python scripts/prof_ops.py $c 1 > gpurun_out/prof_plain_$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"${KRE:-seg_._kernel<\(int\)3}" -c ${NK:-2} \
      -o gpurun_out/gn_${tag}_cfg$c python scripts/prof_ops.py $c 1 > gpurun_out/ncu_gn_$c.log 2>&1
  echo "cfg$c ncu rc=$?"
done
