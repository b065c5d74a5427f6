SKL_NO_PDL=1 timeout 300 python tools/prof_cqr_kernels.py 2048 256 20 1e8 2>&1 | grep -v Warn | tail -22
