#!/bin/bash
# build a tuning variant of the engine: tools/build_var.sh NAME "-DMACRO=V ..." -> lib/var/NAME.so
mkdir -p paper_1405_2636_b200/lib/var
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
  -I include -I paper_1405_2636_b200/csrc $2 -o paper_1405_2636_b200/lib/var/$1.so paper_1405_2636_b200/csrc/ps_b200.cu
