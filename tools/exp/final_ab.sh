for i in 1 2; do
  for c in 0 5; do echo -n "cfg $c "; SRT_PACKET_CFG=$c python tools/time_frames.py 1000000 1920 1080 1 1 20 | grep -o "trace [0-9.]* ms"; done
done
python tools/time_frames.py 100000 512 512 16 1 10 | grep -o "n=.*Msamples/s)"
python tools/time_frames.py 1000000 1920 1080 4 4 5 | grep -o "n=.*Msamples/s)"
python -m pytest tests -m gpu -q -x 2>&1 | tail -1
