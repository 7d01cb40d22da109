#!/bin/bash
# Build an experiment variant of the library: tools/build_variant.sh NAME "-DFIC_TC_XP=..."
set -e
cd /root/repo
# the other objects come from the last in-tree build (run `make` first);
# the variant's source (default fic_tc.cu; SRC=fic_setup.cu ...) is compiled on
# its own so the in-tree library is untouched
SRC=${SRC:-fic_tc.cu}
B=${SRC%.cu}
mkdir -p build/var ab
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr $2 \
  -c paper_1206_4880_b200/csrc/$SRC -o build/var/${B}_$1.o
objs=$(ls build/*.o | grep -v "/$B.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab/$1.so $objs build/var/${B}_$1.o -cudart static
echo built ab/$1.so
