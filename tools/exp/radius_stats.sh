# Per-walk counters of a good (radius 16) and an outlier (radius 12) tree, seed 0, plus the LBVH
for r in 16 12 20; do echo "radius $r: "; SRT_TRACE_STATS=1 SRT_PLOC_RADIUS=$r python tools/time_frames.py 1000000 1920 1080 1 1 3 | grep -o "per walk.*\|trace [0-9.]* ms\|depth': [0-9]*"; done
