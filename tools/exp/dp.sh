echo -n "greedy "; python tools/time_frames.py 1000000 1920 1080 1 1 15 | grep -o "build [0-9.]* ms\|trace [0-9.]* ms" | tr '\n' ' '; echo
for c in "1.0,0.25,1.0" "1.0,0.1,1.0" "1.0,0.5,1.0" "2.0,0.25,1.0" "1.0,0.25,2.0" "0.5,0.25,1.0"; do
  echo -n "dp $c "; SRT_COLLAPSE=dp SRT_COLLAPSE_COSTS=$c python tools/time_frames.py 1000000 1920 1080 1 1 15 | grep -o "build [0-9.]* ms\|trace [0-9.]* ms" | tr '\n' ' '; echo
done
SRT_COLLAPSE=dp python -m pytest tests -m gpu -q -x 2>&1 | tail -1
