# three-way A/B on the C3-target frame: bash tools/exp/ab3.sh A.so B.so C.so
for i in 1 2; do
  for L in "$@"; do echo -n "$(basename $L) "; SRT_LIBSRT_PATH=$L python tools/time_frames.py 1000000 1920 1080 1 1 20 | grep -o "trace [0-9.]* ms"; done
done
