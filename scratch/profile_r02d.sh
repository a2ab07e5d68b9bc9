#!/bin/bash
# Launch lists (ncu gpu__time_duration.sum, cold-cache serialised) of short
# TV / CGLS / SIRT solves at 2048^2 x 1536 on 64 slices, summarised per kernel.
O=gpurun_out
mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/tv3.csv python scratch/tv_probe.py 3 > /dev/null 2>&1
python scratch/tv_launches.py $O/tv3.csv > $O/r02_tv_launches_fused.txt
timeout 600 env ALGO=cgls FILT=none ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/cgls4.csv python scratch/sirt_probe.py 4 > /dev/null 2>&1
python scratch/tv_launches.py $O/cgls4.csv > $O/r02_cgls_launches.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/sirt4.csv python scratch/sirt_probe.py 4 > /dev/null 2>&1
python scratch/tv_launches.py $O/sirt4.csv > $O/r02_sirt_launches.txt
rm -f $O/tv3.csv $O/cgls4.csv $O/sirt4.csv
