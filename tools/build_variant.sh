#!/bin/bash
# Build an experiment variant of the library: tools/build_variant.sh NAME "-DFIC_TC_XP=..."
set -e
cd /root/repo
make -s >/dev/null
mkdir -p build/var
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr $2 \
  -c paper_1206_4880_b200/csrc/fic_tc.cu -o build/var/fic_tc_$1.o
objs=$(ls build/*.o | grep -v fic_tc.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/var/$1.so $objs build/var/fic_tc_$1.o -cudart static
echo built build/var/$1.so
