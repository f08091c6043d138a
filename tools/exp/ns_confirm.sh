python tools/time_frames.py 1000000 1920 1080 4 4 10 | grep -o "n=.*Msamples/s)"
python tools/time_frames.py 1000000 1920 1080 2 2 10 | grep -o "n=.*Msamples/s)"
python tools/time_frames.py 1000000 1920 1080 1 1 20 | grep -o "n=.*Msamples/s)"
python -m pytest tests -m gpu -q -x 2>&1 | tail -1
