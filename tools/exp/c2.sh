python tools/time_frames.py 100000 512 512 1 1 20
python tools/time_frames.py 100000 512 512 16 1 10
python tools/time_frames.py 100000 1024 1024 4 1 10
python tools/time_frames.py 100000 1920 1080 1 1 10
SRT_TRACE_STATS=1 python tools/time_frames.py 100000 512 512 1 1 3 | grep "per walk"
python tools/time_frames.py 1000000 960 540 1 1 20
