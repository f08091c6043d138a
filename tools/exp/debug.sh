# bounds-checked library over the sanitize workload + the GPU parity tests
set -x
SRT_LIBSRT_PATH=paper_2504_06598_b200/libsrt_debug.so timeout 900 python tools/sanitize_workload.py 2>&1 | tail -5
SRT_LIBSRT_PATH=paper_2504_06598_b200/libsrt_debug.so timeout 1500 python -m pytest tests -m gpu -q -x -k "not 6m" 2>&1 | tail -3
python -m pytest tests/test_gpu_parity.py -q -k "render_devices" 2>&1 | tail -2
