for i in 1 2; do
for c in 0 7 8; do echo -n "cfg $c "; SRT_PACKET_CFG=$c python tools/time_frames.py 1000000 1920 1080 4 4 10 | grep -o "trace.*Msamples/s)"; done
done
