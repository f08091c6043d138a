for i in 1 2; do
for c in 0 11 12 13; do echo -n "cfg $c "; SRT_PACKET_CFG=$c python tools/time_frames.py 1000000 1920 1080 1 1 20 | grep -o "trace [0-9.]* ms"; done
done
