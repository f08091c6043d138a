python tools/time_rays.py 1000000 2097152 random 1
python tools/time_rays.py 1000000 2097152 random 4
python tools/time_rays.py 1000000 0 camera 1
SRT_TRACE_VARIANT=0 python tools/time_rays.py 1000000 2097152 random 1
SRT_TRACE_VARIANT=1 python tools/time_rays.py 1000000 2097152 random 1
