# A/B of two libsrt builds on the C3-target frame: bash tools/exp/ab.sh A.so B.so [reps]
A=$1; B=$2
for i in 1 2 3; do
  echo -n "A "; SRT_LIBSRT_PATH=$A python tools/time_frames.py 1000000 1920 1080 1 1 ${3:-20} | grep -o "trace [0-9.]* ms"
  echo -n "B "; SRT_LIBSRT_PATH=$B python tools/time_frames.py 1000000 1920 1080 1 1 ${3:-20} | grep -o "trace [0-9.]* ms"
done
