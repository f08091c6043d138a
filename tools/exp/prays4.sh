# Crossover of sorted packets vs sorted per-lane walks for distinct-origin (parallel jittered) batches
for R in 131072 262144 524288; do
  echo -n "R=$R packets: "; SRT_PACKET_RAYS=1 python tools/time_rays.py 1000000 $R parallel 1 | tail -1
  echo -n "R=$R per-lane: "; SRT_PACKET_RAYS=0 python tools/time_rays.py 1000000 $R parallel 1 | tail -1
done
