#!/bin/bash
# Plain run, launch list, then a full ncu capture of the tensor matcher (1 GPU).
mkdir -p gpurun_out
python tools/prof_encode.py > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_encode.py > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_match_tc -c 1 -o gpurun_out/prof_tc python tools/prof_encode.py > gpurun_out/ncu_full.log 2>&1
echo "profile rc=$?"
