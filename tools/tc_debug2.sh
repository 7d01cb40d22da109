FIC_B200_LIB=build/var/pre.so python tools/gpu_check.py 2>&1 | tail -2
for v in base pre base pre; do echo -n "$v "; FIC_B200_LIB=build/var/$v.so timeout 60 python /tmp/pt.py 2>&1 | tail -1; done
FIC_B200_LIB=build/var/pre.so timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
