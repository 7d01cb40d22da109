# ncu --set full of one k_match_tc launch (cfg3) for the library in $FIC_B200_LIB (default in-tree)
OUT=${1:-gpurun_out/prof_tc}
timeout 120 python tools/prof_encode.py > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_match_tc -c 1 -f -o $OUT python tools/prof_encode.py > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/plain.log
