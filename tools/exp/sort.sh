python -m pytest tests -m gpu -q -x 2>&1 | grep -E "Error|assert|FAILED|Mismatch|passed|failed" | head -5
for v in 0 1; do
  echo "SRT_RAY_SORT=$v"
  SRT_RAY_SORT=$v python tools/time_rays.py 1000000 2097152 random 1
  SRT_RAY_SORT=$v python tools/time_rays.py 1000000 2097152 random 4
  SRT_RAY_SORT=$v python tools/time_rays.py 1000000 0 camera 1
done
