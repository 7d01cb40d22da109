for v in base p4 base p4; do echo -n "$v "; FIC_PLAN_TIMING=1 FIC_B200_LIB=build/var/$v.so timeout 60 python /tmp/pt.py 2>&1 | grep "plan timing" | tail -1 | cut -c1-60; done
