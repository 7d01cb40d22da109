for v in unr um2 um2r1 unr um2 um2r1; do echo -n "$v "; FIC_B200_LIB=build/var/$v.so timeout 60 python /tmp/pt.py 2>&1 | tail -1; done
