for v in n128 n256 n128 n256; do echo "$v"; FIC_B200_LIB=build/var/$v.so timeout 60 python tools/prof_encode.py 2>&1 | tail -1; done
FIC_B200_LIB=build/var/n256.so timeout 120 python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | cut -c1-250
