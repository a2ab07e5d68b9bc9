#!/bin/bash
# Round profiling pass (run under gpurun): launch list of the bench step and
# ncu --set full captures of the hot kernels.  Outputs in gpurun_out/.
set -x
O=gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for k in ${KERNELS:-k_spmm k_sh_tma k_fft1_fwd_pers k_fft1_inv_pers k_fft2_col_pers k_fft2_row_unpack_pers k_fft2_row_pack_pers}; do
  REPS=1 timeout 400 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^$k" -s 2 -c 1 -o $O/full_$k python scratch/op_probe.py > $O/full_$k.log 2>&1
done
