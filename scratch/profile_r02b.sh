#!/bin/bash
# Second round-2 capture set: the spectral reduction and the TV / CGLS passes
# (demangled-name regexes), summarised on the box.
O=gpurun_out
timeout 400 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"k_spec<float, float2, 0>" -s 2 -c 1 -o $O/r02_full_k_spec python scratch/sirt_probe.py 3 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"k_spec<float, float2, 1>" -c 1 -o $O/r02_full_k_spec_update python scratch/tv_probe.py 1 > /dev/null 2>&1
for k in OpTvStepS OpTvShrink "OpTvS<float, 2" "OpTvS<float, 0" OpTvGradNorm; do
  n=$(echo "$k" | tr -dc 'A-Za-z0-9')
  timeout 400 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:$k" -c 1 -o $O/r02_full_$n python scratch/tv_probe.py 1 > /dev/null 2>&1
done
ALGO=cgls FILT=none timeout 400 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"OpCglsTail" -c 1 -o $O/r02_full_OpCglsTail python scratch/sirt_probe.py 3 > /dev/null 2>&1
ON_BOX=1 python scratch/summarize_r02.py > /dev/null 2>&1
mv $O/r02_ncu_full_summary.txt $O/r02_ncu_full_summary_solvers.txt
rm -f $O/r02_full_*.ncu-rep
