export SRT_LIBSRT_PATH=paper_2504_06598_b200/libsrt_exp.so
for C in 0 2 3; do echo "C2 C=$C: $(SRT_SPLIT_CELLS=$C timeout 300 python tools/time_frames.py 100000 512 512 16 1 10 2>&1 | tail -1 | cut -c1-110)"; done
for C in 0 2; do echo "C2 1spp C=$C: $(SRT_SPLIT_CELLS=$C timeout 300 python tools/time_frames.py 100000 512 512 1 1 20 2>&1 | tail -1 | cut -c1-110)"; done
for C in 0 7; do echo "1M 16spp C=$C: $(SRT_SPLIT_CELLS=$C timeout 300 python tools/time_frames.py 1000000 1920 1080 16 1 5 2>&1 | tail -1 | cut -c1-110)"; done
for C in 0 7; do echo "1M 1spp C=$C: $(SRT_SPLIT_CELLS=$C timeout 300 python tools/time_frames.py 1000000 1920 1080 1 1 10 2>&1 | tail -1 | cut -c1-110)"; done
