#!/bin/bash
# K1 timing of library variants: tools/ab_pool.sh cfg3 cfg5 -- vlib/a.so vlib/b.so
cfgs=(); while [ "$1" != "--" ]; do cfgs+=("$1"); shift; done; shift
for r in 1 2; do for L in "$@"; do FIC_B200_LIB=$L python tools/pool_time.py "${cfgs[@]}" | sed "s|^|$(basename $L) |"; done; done
