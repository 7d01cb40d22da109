#!/bin/bash
# One profiling round on one GPU (all logs under gpurun_out/): the bench line,
# K1 alone, launch lists of one encode per config, and ncu --set full
# captures of the top kernels (each only after its command ran clean without ncu).
mkdir -p gpurun_out
set -x
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python tools/pool_time.py cfg3 cfg5 > gpurun_out/pool_time.log 2>&1
for c in cfg3 cfg4 cfg5; do
  timeout 300 python tools/prof_encode.py $c > gpurun_out/plain_$c.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$c.csv python tools/prof_encode.py $c > gpurun_out/ncu_launch_$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_match_tc|k_pool|k_fd16|k_domrows" -c 4 \
  -o gpurun_out/prof_cfg3 python tools/prof_encode.py cfg3 > gpurun_out/ncu_full_cfg3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_match_tc|k_hl_rescore" -c 2 \
  -o gpurun_out/prof_cfg4 python tools/prof_encode.py cfg4 > gpurun_out/ncu_full_cfg4.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_fd16|k_pool|k_boxplanes" -c 3 \
  -o gpurun_out/prof_cfg5 python tools/prof_encode.py cfg5 > gpurun_out/ncu_full_cfg5.log 2>&1
echo done
