for i in 1 2 3; do python tools/prof_qr.py 8192 1024 3; python tools/prof_qr.py 2048 257 3; done
python tools/time_solve.py 2
