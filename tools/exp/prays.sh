# Explicit-ray routes: packets (auto) vs per-lane walks (SRT_PACKET_RAYS=0), 1M cloud
for k in camera parallel random; do
  for pr in -1 0; do echo -n "SRT_PACKET_RAYS=$pr "; SRT_PACKET_RAYS=$pr python tools/time_rays.py 1000000 2097152 $k 1 | tail -1; done
done
echo -n "camera N=4 packets: "; python tools/time_rays.py 1000000 2097152 camera 4 | tail -1
echo -n "camera N=4 per-lane: "; SRT_PACKET_RAYS=0 python tools/time_rays.py 1000000 2097152 camera 4 | tail -1
