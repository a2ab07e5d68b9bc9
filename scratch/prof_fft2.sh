O=gpurun_out
for k in k_fft2_col k_fft2_row_unpack; do
  REPS=1 timeout 400 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^$k" -s 1 -c 1 -o $O/full_$k python scratch/op_probe.py > $O/full_$k.log 2>&1
done
