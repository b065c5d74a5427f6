python tools/time_solve.py 2
python tools/time_solve.py 1
for mn in "800 201" "2048 257"; do
  python tools/prof_qr.py $mn 3
  SKL_QR_BLOCKED_MIN_N=100000 python tools/prof_qr.py $mn 3
done
