#!/bin/bash
# One GPU round trip: bring-up check, gpu tests, bench.  Logs in gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/check.log 2>&1
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
fi
timeout 300 python bench.py --steps 5 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
cat gpurun_out/check.log; tail -4 gpurun_out/pytest_gpu.log 2>/dev/null
python - <<'PY'
import json
for l in open('gpurun_out/bench.log'):
    if l.startswith('{'):
        d=json.loads(l); print('value %.4g ms %.3f frac %.3f e2e %.4g' % (d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])); print(d['device_stats'], d.get('clocks'))
    else: print(l.rstrip())
PY
