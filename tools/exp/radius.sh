for r in 8 12 16 20 24; do echo -n "radius $r: "; SRT_PLOC_RADIUS=$r python tools/time_frames.py 1000000 1920 1080 1 1 15 | grep -o "build.*ms  n\|trace [0-9.]* ms"| tr '\n' ' '; echo; done
