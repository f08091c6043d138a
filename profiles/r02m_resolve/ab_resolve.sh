timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/resolve_tests.txt 2>&1; tail -2 gpurun_out/resolve_tests.txt
for L in build/ab/libsrt_prev.so paper_2504_06598_b200/libsrt.so; do echo $L; SRT_LIBSRT_PATH=$L timeout 600 python tools/time_render_configs.py 2>&1 | grep render; done
