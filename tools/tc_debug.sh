FIC_TC_DEBUG=40 timeout 60 python tools/prof_encode.py 2>&1 | tail -22
