# Incoherent (random) explicit rays: sorted packets (SRT_PACKET_RAYS=1) vs per-lane / coop walks
for N in 1 4; do
  for pr in 1 0; do echo -n "SRT_PACKET_RAYS=$pr "; SRT_PACKET_RAYS=$pr python tools/time_rays.py 1000000 2097152 random $N | tail -1; done
done
echo -n "unsorted packets: "; SRT_RAY_SORT=0 SRT_PACKET_RAYS=1 python tools/time_rays.py 1000000 2097152 random 1 | tail -1
