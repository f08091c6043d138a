# Grid resolution of the split tree by scene size (experiments build).
mkdir -p gpurun_out
export SRT_LIBSRT_PATH=paper_2504_06598_b200/libsrt_exp.so
{
for C in 4 6 7 8; do echo "1M C=$C $(SRT_SPLIT_CELLS=$C timeout 300 python tools/ab_frames.py 15 2>&1 | grep mean)"; done
for C in 0 2 3 4; do echo "100k 512 C=$C $(SRT_N=100000 SRT_W=512 SRT_H=512 SRT_SPLIT_CELLS=$C timeout 300 python tools/ab_frames.py 20 0 1 2>&1 | grep mean)"; done
for C in 0 4 6 8 10; do echo "3M 4K C=$C $(SRT_N=3000000 SRT_W=3840 SRT_H=2160 SRT_SPLIT_CELLS=$C timeout 300 python tools/ab_frames.py 10 0 2>&1 | grep mean)"; done
for C in 0 6 8 10 12; do echo "6M C=$C $(SRT_N=6000000 SRT_SPLIT_CELLS=$C timeout 300 python tools/ab_frames.py 10 0 2>&1 | grep mean)"; done
} > gpurun_out/split_sizes.txt 2>&1
cat gpurun_out/split_sizes.txt
