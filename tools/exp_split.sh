# Split-tree experiments on a GPU box (outputs in gpurun_out/): the GPU tests,
# frame times for several grid resolutions, explicit-ray throughput.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/split_tests.txt 2>&1; tail -5 gpurun_out/split_tests.txt
export SRT_LIBSRT_PATH=paper_2504_06598_b200/libsrt_exp.so
for C in ${CELLS:-3 4 5 6}; do SRT_SPLIT_CELLS=$C timeout 300 python tools/ab_frames.py 15 2>&1 | grep mean; done > gpurun_out/split_ab2.txt
cat gpurun_out/split_ab2.txt
for C in 0 4; do for k in "random 1" "random 4" "camera 1"; do echo "C=$C $k: $(SRT_SPLIT_CELLS=$C timeout 300 python tools/time_rays.py 1000000 2097152 $k 2>&1 | tail -1)"; done; done > gpurun_out/split_rays.txt
cat gpurun_out/split_rays.txt
