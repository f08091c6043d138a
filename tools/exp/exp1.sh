python -m pytest tests/test_gpu_parity.py -q -k mapped 2>&1 | tail -2
python tools/time_frames.py 1000000 1920 1080 1 1 20
SRT_TRACE_STATS=1 python tools/time_frames.py 1000000 1920 1080 1 1 3 | grep "per walk"
SRT_SAH=1 SRT_SAH_TIGHT=1 SRT_SAH_LEAF=1 python tools/time_frames.py 1000000 1920 1080 1 1 20
SRT_SAH=1 SRT_SAH_TIGHT=1 SRT_SAH_LEAF=1 SRT_TRACE_STATS=1 python tools/time_frames.py 1000000 1920 1080 1 1 3 | grep "per walk"
SRT_PACKET_CFG=3 python tools/time_frames.py 1000000 1920 1080 1 1 20
python tools/time_frames.py 1000000 1920 1080 4 4 10
python tools/time_frames.py 100000 512 512 16 1 10
python tools/time_frames.py 3000000 3840 2160 4 1 5
python tools/time_frames.py 6000000 1920 1080 1 1 10
