timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_gpu_packet_rays.py -x -q > gpurun_out/exact_tests.txt 2>&1; tail -2 gpurun_out/exact_tests.txt
for L in build/ab/libsrt_prev.so paper_2504_06598_b200/libsrt.so build/ab/libsrt_prev.so paper_2504_06598_b200/libsrt.so; do echo $L; SRT_LIBSRT_PATH=$L timeout 600 python tools/time_paths.py 2>&1 | grep -E "exact|biased"; done
