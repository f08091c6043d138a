python -m pytest tests/test_gpu_parity.py -q -k "degenerate" 2>&1 | tail -2
for v in 0 1 2; do
  echo "variant $v"
  SRT_TRACE_VARIANT=$v python tools/time_rays.py 1000000 2097152 random 1
  SRT_TRACE_VARIANT=$v python tools/time_rays.py 1000000 0 camera 1
  SRT_TRACE_VARIANT=$v python tools/time_rays.py 1000000 2097152 random 4
done
