#!/bin/bash
# Interleaved comparison of several library builds on cfg3 (ms_tensor):
#   tools/ab_multi.sh ROUNDS lib1.so lib2.so ...
N=$1; shift
for i in $(seq $N); do
  for L in "$@"; do
    FIC_B200_LIB=$L timeout 60 python tools/seg_sweep.py 131072 2>&1 | tail -1 | sed "s|^|$(basename $L) |"
  done
done
