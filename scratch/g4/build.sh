#!/bin/bash
cd "$(dirname "$0")" && /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -shared -Xcompiler -fPIC -o libg4.so g4.cu -lcuda
