for args in "100000 512 512 16 1 10" "1000000 1920 1080 16 1 5" "6000000 1920 1080 16 1 5" "3000000 3840 2160 4 1 5"; do
  for L in build/ab/libsrt_head.so build/ab/libsrt_pm.so; do
    echo -n "$(basename $L) "; SRT_LIBSRT_PATH=$L SRT_ONE_LAUNCH=1 python tools/time_frames.py $args | grep -o "n=.*Msamples/s)"
  done
done
python -m pytest tests -m gpu -q -x -k "one_launch or render_devices or distributed or mapped or a06 or a10" 2>&1 | tail -1
