# PLOC neighbourhood radius on the split tree (experiments build, SRT_PLOC_RADIUS).
export SRT_LIBSRT_PATH=paper_2504_06598_b200/libsrt_exp.so
for R in 16 8 12 24 32 16; do echo "radius $R: $(SRT_PLOC_RADIUS=$R timeout 300 python tools/ab_frames.py 15 2>&1 | grep mean)"; done
