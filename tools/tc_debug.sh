for cg in 1 2; do FIC_TC_CG=$cg timeout 60 python tools/prof_encode.py; FIC_TC_CG=$cg timeout 60 python tools/prof_encode.py; done
