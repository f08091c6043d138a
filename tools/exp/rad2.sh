for r in 12 16 24 32; do echo -n "radius $r: "; SRT_PLOC_RADIUS=$r SRT_TRACE_STATS=1 python tools/time_frames.py 1000000 1920 1080 1 1 3 | grep -o "per walk.*\|depth': [0-9]*" | tr '\n' ' '; echo; done
for r in 12 16 24; do echo -n "radius $r 100k: "; SRT_PLOC_RADIUS=$r python tools/time_frames.py 100000 1920 1080 1 1 10 | grep -o "trace [0-9.]* ms\|depth': [0-9]*" | tr '\n' ' '; echo; done
