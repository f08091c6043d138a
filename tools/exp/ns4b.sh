for i in 1 2; do
for c in 0 14 15; do echo -n "N=4 cfg $c "; SRT_PACKET_CFG=$c python tools/time_frames.py 1000000 1920 1080 4 4 10 | grep -o "trace.*Msamples/s)"; done
for c in 0 14 15; do echo -n "N=2 cfg $c "; SRT_PACKET_CFG=$c python tools/time_frames.py 1000000 1920 1080 2 2 10 | grep -o "trace.*Msamples/s)"; done
done
