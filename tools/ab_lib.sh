#!/bin/bash
# A/B of two library builds on cfg3, alternating processes:
#   tools/ab_lib.sh A.so B.so [rounds]
A=$1; B=$2; N=${3:-4}
for i in $(seq $N); do
  for L in $A $B; do
    FIC_B200_LIB=$L python tools/seg_sweep.py 131072 2>&1 | sed "s|^|$(basename $L) |"
  done
done
