#!/bin/bash
# build_variant.sh NAME "-DFLAG=.. ..."  -> paper_2003_12677_b200/NAME.so (tuning experiments)
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
OUT=/tmp/var_$NAME; mkdir -p $OUT
for f in paper_2003_12677_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --expt-relaxed-constexpr -Xcompiler -fPIC -I include $@ -c $f -o $OUT/$(basename $f .cu).o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2003_12677_b200/$NAME.so $OUT/*.o -L /usr/local/cuda/lib64 -lcufft -Xlinker -rpath,/usr/local/cuda/lib64
