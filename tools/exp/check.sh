# GPU tests (product lib), debug-lib workload, and the bench line
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
SRT_LIBSRT_PATH=paper_2504_06598_b200/libsrt_debug.so timeout 900 python tools/sanitize_workload.py 2>&1 | tail -2
python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | tail -1
