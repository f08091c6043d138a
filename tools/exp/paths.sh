python tools/time_paths.py 2>&1 | grep -v Warn
SRT_ONE_LAUNCH=1 python tools/time_frames.py 6000000 1920 1080 1024 1 2 | grep -o "n=.*Msamples/s)"
