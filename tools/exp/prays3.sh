# Packets from distinct origins below the per-lane sort threshold (sorted since this change) vs per-lane
for R in 16384 60000; do
  echo -n "R=$R packets: "; python tools/time_rays.py 1000000 $R parallel 1 | tail -1
  echo -n "R=$R per-lane: "; SRT_PACKET_RAYS=0 python tools/time_rays.py 1000000 $R parallel 1 | tail -1
done
