# End-of-round evidence on one GPU box (outputs in gpurun_out/, TAG prefix):
# GPU tests, the measure.sh set (bench line, reference arm, launch list, ncu
# full of k_trace_packet), scene seeds, secondary paths, BASELINE configs,
# explicit rays, tile-shard bounds.
mkdir -p gpurun_out
TAG=${TAG:-r02h}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.txt 2>&1; tail -2 gpurun_out/${TAG}_gpu_tests.txt
TAG=$TAG bash tools/measure.sh > gpurun_out/${TAG}_measure.log 2>&1; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-200
timeout 300 python tools/ab_frames.py 20 > gpurun_out/${TAG}_seeds.log 2>&1; tail -1 gpurun_out/${TAG}_seeds.log
timeout 900 python tools/time_paths.py > gpurun_out/${TAG}_paths.log 2>&1; tail -12 gpurun_out/${TAG}_paths.log
{
echo "C2 100k 512x512 16spp N=1: $(timeout 300 python tools/time_frames.py 100000 512 512 16 1 10 2>&1 | tail -1)"
echo "C3 1M 1080p 1spp N=4: $(timeout 300 python tools/time_frames.py 1000000 1920 1080 1 4 10 2>&1 | tail -1)"
echo "1M 1080p 1spp N=8: $(timeout 300 python tools/time_frames.py 1000000 1920 1080 1 8 10 2>&1 | tail -1)"
echo "1M 1080p 16spp N=1: $(timeout 300 python tools/time_frames.py 1000000 1920 1080 16 1 5 2>&1 | tail -1)"
echo "C4 3M 3840x2160 4spp N=1: $(timeout 300 python tools/time_frames.py 3000000 3840 2160 4 1 5 2>&1 | tail -1)"
echo "6M 1080p 1spp N=1: $(timeout 300 python tools/time_frames.py 6000000 1920 1080 1 1 10 2>&1 | tail -1)"
echo "C5 6M 1080p 1024spp N=1: $(timeout 600 python tools/time_frames.py 6000000 1920 1080 1024 1 2 2>&1 | tail -1)"
} > gpurun_out/${TAG}_configs.log 2>&1; cat gpurun_out/${TAG}_configs.log
{
for k in "random 1" "random 4" "camera 1" "camera 4" "parallel 1"; do echo "$k: $(timeout 300 python tools/time_rays.py 1000000 2097152 $k 2>&1 | tail -1)"; done
} > gpurun_out/${TAG}_rays.log 2>&1; cat gpurun_out/${TAG}_rays.log
timeout 300 python tools/shard_times.py 0 > gpurun_out/${TAG}_shards.log 2>&1; tail -4 gpurun_out/${TAG}_shards.log
timeout 300 python tools/shard_times.py 0 3000000 3840 2160 > gpurun_out/${TAG}_shards_c4.log 2>&1; tail -4 gpurun_out/${TAG}_shards_c4.log
