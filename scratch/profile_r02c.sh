#!/bin/bash
O=gpurun_out
timeout 400 ncu --set full --clock-control none --kernel-name-base function -k regex:"^k_spec" -s 2 -c 1 -o $O/r02_full_k_spec python scratch/sirt_probe.py 3 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:k_spec<float, float2, (true|1|\(bool\)1)>" -c 1 -o $O/r02_full_k_spec_update python scratch/tv_probe.py 1 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:OpTvS<float, (2|\(int\)2)" -c 1 -o $O/r02_full_OpTvS2 python scratch/tv_probe.py 1 > /dev/null 2>&1
ON_BOX=1 python scratch/summarize_r02.py > /dev/null 2>&1
mv $O/r02_ncu_full_summary.txt $O/r02_ncu_full_summary_spec.txt
ncu --query-metrics > /dev/null 2>&1
rm -f $O/r02_full_*.ncu-rep
