python tools/gpu_check.py 2>&1 | tail -3
FIC_PLAN_TIMING=1 python /tmp/pt.py 2>&1 | tail -2
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
