python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for N in 4 8 16; do python tools/time_frames.py 1000000 1920 1080 $N $N 5 | grep -o "n=.*Msamples/s)"; done
python tools/time_frames.py 1000000 1920 1080 1 1 20 | grep -o "n=.*Msamples/s)"
