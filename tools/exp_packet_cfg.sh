# Packet-kernel batch / occupancy configurations on the split tree (experiments build, SRT_PACKET_CFG).
export SRT_LIBSRT_PATH=paper_2504_06598_b200/libsrt_exp.so
for c in 0 1 2 3 12 13 0; do echo "cfg $c: $(SRT_PACKET_CFG=$c timeout 300 python tools/ab_frames.py 15 2>&1 | grep mean)"; done
