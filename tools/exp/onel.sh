python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for args in "100000 512 512 16 1 10" "100000 1024 1024 4 1 10" "1000000 1920 1080 4 4 10" "1000000 960 540 1 1 20" "3000000 3840 2160 4 1 5" "1000000 1920 1080 1 1 20"; do
  echo -n "per-pass:  "; python tools/time_frames.py $args | grep -o "n=.*Msamples/s)"
  echo -n "one-launch: "; SRT_ONE_LAUNCH=1 python tools/time_frames.py $args | grep -o "n=.*Msamples/s)"
done
