#!/bin/bash
# Round-2 profiling pass (run under gpurun): launch list of the bench's
# gridrec step and ncu --set full captures of the hot kernels (one launch
# each) -- gridrec / radon operators, the SIRT spectral reduction, the TV
# element passes.  Outputs in gpurun_out/.
O=gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/r02_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-parity --no-solvers --pipeline-slices 0 > /dev/null 2>&1
for k in k_spmm_seg k_sh_tma k_fft1_fwd_pers k_fft1_inv_pers k_fft2_col_pers k_fft2_row_unpack_pers k_fft2_row_pack_pers; do
  REPS=1 timeout 400 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^$k" -s 2 -c 1 -o $O/r02_full_$k python scratch/op_probe.py > /dev/null 2>&1
done
timeout 400 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_spec<float, float2, false>" -s 2 -c 1 -o $O/r02_full_k_spec python scratch/sirt_probe.py 3 > /dev/null 2>&1
for k in OpTvStep OpTvShrink "OpTvS<float, 2" OpTvGradNorm; do
  n=$(echo "$k" | tr -dc 'A-Za-z0-9')
  timeout 400 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$k" -c 1 -o $O/r02_full_$n python scratch/tv_probe.py 1 > /dev/null 2>&1
done
ls $O/r02_full_* > $O/r02_profile_done.txt
# summaries travel back (gpurun_out is capped at 64 MiB): keep the text, the
# launch list and the S kernel's report only
ON_BOX=1 python scratch/summarize_r02.py > /dev/null 2>&1
python scratch/ncu_summary.py $O/r02_launches_bench.csv > $O/r02_launches_bench_summary.txt 2>&1
for f in $O/r02_full_*.ncu-rep; do
  case "$f" in *k_spmm_seg*) ;; *) rm -f "$f" ;; esac
done
