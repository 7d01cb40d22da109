FIC_B200_LIB=build/var/win.so python tools/gpu_check.py 2>&1 | tail -2
for v in base win base win; do echo -n "$v "; FIC_B200_LIB=build/var/$v.so timeout 60 python /tmp/pt.py 2>&1 | tail -1; done
